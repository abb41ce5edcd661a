"""The reference-side C++ binding (include/qweight_b200.hpp) on the GPU.

tests/native/shim_gpu.cpp is built by oracle/Makefile (here, where the
reference's headers exist) against the reference's own library and
libqweight_b200.so, and ships prebuilt to the GPU box like oracle/_ref.  It
quantizes a layer with the reference's synth + quantize_layer, runs it through
qweight::b200::DeviceLayer / matvec_pipelined / bench_matvec, and checks it
with the reference's own reconstruct_dense (bit for bit) and
matvec_reference_f64 (1e-2), plus the reference's error contract."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SHIM = ROOT / "oracle" / "_ref" / "shim_gpu"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not SHIM.exists(), reason="shim_gpu not built (needs the reference headers at build time)")
@pytest.mark.parametrize("rows,cols", [(1024, 4096), (4096, 4096), (4096, 11008)])
def test_cpp_shim_on_gpu(rows, cols):
    out = subprocess.run([str(SHIM), str(rows), str(cols)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    kv = dict(line.split(" ", 1) for line in out.stdout.splitlines() if " " in line and not line.startswith("rows,"))
    assert float(kv["rel_l2"]) <= 1e-2
    assert kv["fails"] == "0"
