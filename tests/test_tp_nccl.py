"""The C-ABI tensor-parallel entries (include/qweight_b200_tp.h,
libqweight_b200_tp.so) on a real NCCL communicator.  This box has one GPU,
so the communicator has one rank (ncclCommInitAll over device 0): the shard
+ collective + unpad / gather kernels all run, the exchange is trivial.  The
multi-rank split logic is covered by tests/test_tp.py (gloo, 2 and 4 ranks,
also on the GPU)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw

pytestmark = pytest.mark.gpu
TP_LIB = Path(qw.__file__).resolve().parent / "lib" / "libqweight_b200_tp.so"


def _nccl_comm():
    nccl = C.CDLL("libnccl.so.2")
    comm = C.c_void_p()
    devs = (C.c_int * 1)(0)
    assert nccl.ncclCommInitAll(C.byref(comm), 1, devs) == 0
    return nccl, comm


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("batch", [1, 4])
def test_tp_c_abi_single_rank_nccl(mode, batch):
    import torch
    qw.lib()  # the main library first (the TP library links it)
    tp_lib = C.CDLL(str(TP_LIB))
    nccl, comm = _nccl_comm()
    layer = qw.synth_layer(384, 1024, seed=91, outlier_ratio=0.005)
    h = layer._handle()
    tp = C.c_void_p()
    try:
        assert tp_lib.qw_tp_create(h, 0, 1, mode, 0, 0, C.byref(tp)) == 0
    finally:
        qw.lib().qw_host_free(h)
    xs = np.stack([qw.synth_activation(1024, 92 + b) for b in range(batch)])
    x = torch.from_numpy(xs).cuda()
    y = torch.empty(batch, 384, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    assert tp_lib.qw_tp_matvec(tp, C.c_void_p(x.data_ptr()), batch, C.c_void_p(y.data_ptr()), comm,
                               C.c_void_p(stream)) == 0
    torch.cuda.synchronize()
    for b in range(batch):
        ref = oracle.matvec_f64(layer, xs[b])
        assert np.linalg.norm(y[b].cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-2
    rows, cols = C.c_uint32(), C.c_uint32()
    assert tp_lib.qw_tp_local_extent(tp, C.byref(rows), C.byref(cols)) == 0
    assert rows.value == 384
    tp_lib.qw_tp_free(tp)
    nccl.ncclCommDestroy(comm)


@pytest.mark.parametrize("mode", [0, 1])
def test_tp_c_abi_peer_exchange_single_rank(mode):
    """qw_tp_bind_peers / qw_tp_matvec_peer: the exchange fused with the GEMV
    over peer memory, one rank (it pushes into its own buffer and waits for
    its own arrivals; the multi-rank protocol is tests/test_tp.py), twice."""
    import torch
    qw.lib()
    tp_lib = C.CDLL(str(TP_LIB))
    layer = qw.synth_layer(384, 1024, seed=93, outlier_ratio=0.005)
    h = layer._handle()
    tp = C.c_void_p()
    try:
        assert tp_lib.qw_tp_create(h, 0, 1, mode, 0, 2, C.byref(tp)) == 0  # QW_UPLOAD_SIMT
    finally:
        qw.lib().qw_host_free(h)
    nbytes = C.c_uint64()
    assert tp_lib.qw_tp_exchange_bytes(tp, C.byref(nbytes)) == 0
    buf = torch.zeros(nbytes.value // 4, dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    arrivals = tp_lib.qw_tp_arrivals(tp)
    assert arrivals > 0
    bufs = (C.c_void_p * 1)(buf.data_ptr())
    flags = (C.c_void_p * 1)(flag.data_ptr())
    assert tp_lib.qw_tp_bind_peers(tp, bufs, flags, arrivals) == 0
    for k in range(2):
        x = torch.from_numpy(qw.synth_activation(1024, 94 + k)).cuda()
        y = torch.empty(384, device="cuda")
        assert tp_lib.qw_tp_matvec_peer(tp, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        torch.cuda.synchronize()
        ref = oracle.matvec_f64(layer, qw.synth_activation(1024, 94 + k))
        assert np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref) <= 1e-2
        assert int(flag.item()) == 0
    tp_lib.qw_tp_free(tp)
