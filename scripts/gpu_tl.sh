cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
QW_PLAN_DEBUG=1 python -c "
import sys; sys.path.insert(0,'.')
import paper_2311_16442_b200 as qw
for r,c,ratio in [(5120,13824,0.01),(13824,5120,0.01),(8192,28672,0.002)]:
    qw.DeviceLayer(qw.synth_layer(r,c,seed=7,outlier_ratio=ratio))
" 2>&1 | grep "qw plan"
