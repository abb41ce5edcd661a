"""BASELINE config 5: Llama-2-70B linear shapes, column/row tensor-parallel split
at N = WORLD_SIZE GPUs over NCCL (launch with torchrun).  Per shape: local GEMV
us, collective us, end-to-end us -- each the max over ranks, CUDA events.
usage: torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/tp_bench.py"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200.tp import TPLinear  # noqa: E402

SHAPES = [("q_o", 8192, 8192, "col"), ("kv", 1024, 8192, "col"), ("gate_up", 28672, 8192, "col"),
          ("down", 8192, 28672, "row"), ("o_row", 8192, 8192, "row")]
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{local}"))
cache = Path(os.environ.get("QW_BENCH_CACHE", "/tmp/qw_bench_cache"))
cache.mkdir(parents=True, exist_ok=True)


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


for name, rows, cols, mode in SHAPES:
    path = cache / f"llama70b_{rows}x{cols}.qwl"
    if rank == 0 and not path.exists():  # quantize the whole layer once, then shard
        qw.write_packed_layer(qw.synth_layer(rows, cols, seed=7), str(path) + ".tmp")
        os.replace(str(path) + ".tmp", path)
    dist.barrier()
    layer = qw.read_packed_layer(str(path))
    tp = TPLinear(layer, rank, world, mode, device=f"cuda:{local}")
    x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
    if mode == "row":
        xs = (x.index_select(0, tp.gidx) * tp.gmask).contiguous()
        y_loc = torch.empty(tp.shard.cfg.rows, device="cuda")
        us_gemv = timed(lambda: tp.dl.matvec(xs, out=y_loc))
        us_coll = timed(lambda: dist.all_reduce(y_loc))
    else:
        y_loc = torch.empty(tp.shard.cfg.rows, device="cuda")
        us_gemv = timed(lambda: tp.dl.matvec(x, out=y_loc))
        buf = torch.zeros(tp.max_rows, device="cuda")
        out = torch.empty(world * tp.max_rows, device="cuda")
        us_coll = timed(lambda: dist.all_gather_into_tensor(out, buf))
    us_e2e = timed(lambda: tp.forward(x))
    y = tp.forward(x)
    if rank == 0:
        import oracle
        ref = oracle.matvec_f64(layer, qw.synth_activation(cols, 8))
        rel = float(np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref))
        bal = qw.payload_bytes(layer) + 4 * (rows + cols)
        print(json.dumps({"shape": name, "rows": rows, "cols": cols, "mode": mode, "n_gpus": world,
                          "us_gemv": round(us_gemv, 3), "us_collective": round(us_coll, 3),
                          "us_end_to_end": round(us_e2e, 3),
                          "gb_s_end_to_end": round(bal / us_e2e / 1e3, 1), "rel_l2_vs_f64": rel}),
              flush=True)
dist.destroy_process_group()
