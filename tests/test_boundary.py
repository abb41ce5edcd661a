"""The drop-in boundary, checked without a GPU.

  * libqweight_b200.so exports every entry point include/qweight_b200.h
    declares (the C-ABI a reference-side binding links against);
  * the C++ shim include/qweight_b200.hpp compiles and links against the
    reference's own headers (proj/include/qweight/*.hpp), i.e. the
    reference's API types go straight in (skipped where /root/reference is
    absent, e.g. on the GPU box);
  * status codes and messages behave like qweight::Error on bad input.
"""
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2311_16442_b200 as qw
from paper_2311_16442_b200 import _native

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "qweight_b200.h"
REF_INC = Path("/root/reference/proj/include")


def declared_functions() -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return set(re.findall(r"\b(qw_[a-z0-9_]+)\s*\(", text))


def exported_dynamic() -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.lib_path())],
                         capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


def test_every_declared_entry_point_is_exported():
    declared = declared_functions()
    assert len(declared) >= 30
    missing = declared - exported_dynamic()
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert declared_functions() <= set(qw.exported_symbols())


def test_abi_version_and_strerror():
    L = qw.lib()
    assert L.qw_abi_version() == 1
    assert L.qw_strerror(0) == b"ok"
    assert L.qw_strerror(2) == b"invalid layer"
    assert L.qw_strerror(99) == b"unknown status"


def test_null_handles_are_argument_errors_without_a_device():
    """The ABI never dereferences a null handle: every entry that takes one
    returns QW_ERR_ARG (status 1) before touching CUDA."""
    import ctypes as C
    L = qw.lib()
    null = C.c_void_p()
    outs = (C.c_void_p * 1)()
    assert L.qw_group_matvec(null, null, outs, null, 0) == 1
    assert L.qw_group_matvec_batch(null, null, 2, outs, null, 0) == 1
    assert L.qw_matvec_uses_gemm(null, 4, 0) == -1  # (0 / 1 are answers)
    assert L.qw_matvec_ex(null, null, 1, null, null, null, 0) == 1


def test_invalid_view_is_rejected_with_layer_status():
    import dataclasses
    layer = qw.synth_layer(8, 64, seed=1)
    bad = dataclasses.replace(layer, meta=layer.meta[:-1])
    with pytest.raises(qw.QWeightError) as ei:
        qw.validate_layer(bad)
    assert ei.value.status == 2


@pytest.mark.skipif(not REF_INC.exists() or shutil.which("g++") is None,
                    reason="reference headers not present (GPU box)")
def test_cpp_shim_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "shim.cpp"
    src.write_text(
        '#include "qweight_b200.hpp"\n'
        "int main() {\n"
        "  qweight::PackedLayer L;\n"
        "  try { qweight::b200::matvec_pipelined(L, std::span<const float>{}, 0); }\n"
        "  catch (const qweight::Error&) { return qw_abi_version() == 1 ? 0 : 2; }\n"
        "  return 1;\n"
        "}\n")
    exe = tmp_path / "shim"
    lib_dir = _native.lib_path().parent
    subprocess.run(["g++", "-std=c++20", f"-I{REF_INC}", f"-I{ROOT / 'include'}", str(src),
                    f"-L{lib_dir}", "-lqweight_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
                   check=True)
    # workers == 0 throws qweight::Error before touching the device (engine.cpp:187-188)
    assert subprocess.run([str(exe)]).returncode == 0


def test_diagnostic_knobs_are_inert_without_the_debug_gate():
    """The library reads its diagnostic knobs (QW_NQ1, QW_GEMM_KS, ...) only
    under QW_DEBUG_KNOBS=1: the product's behaviour never depends on the
    environment.  Checked in fresh processes."""
    import os
    import subprocess
    import sys
    code = ("import paper_2311_16442_b200 as qw; L = qw.lib(); "
            "print(L.qw_debug_knob(b'QW_NQ1', 2), L.qw_debug_knob(b'QW_GEMM_KS', 0), "
            "L.qw_debug_knob(b'QW_TEAMS_MIN_NQ', 4))")
    env = {k: v for k, v in os.environ.items() if k != "QW_DEBUG_KNOBS"}
    env.update(QW_NQ1="1", QW_GEMM_KS="3", QW_TEAMS_MIN_NQ="9")
    run = lambda e: subprocess.run([sys.executable, "-c", code], env=e, cwd=str(ROOT), capture_output=True,  # noqa: E731
                                   text=True, check=True).stdout.split()
    assert run(env) == ["2", "0", "4"]          # defaults pinned
    assert run({**env, "QW_DEBUG_KNOBS": "1"}) == ["1", "3", "9"]  # the gate opens them


def test_tp_library_exports_its_header():
    """include/qweight_b200_tp.h <-> libqweight_b200_tp.so (NCCL and peer-exchange entries)."""
    tp_h = ROOT / "include" / "qweight_b200_tp.h"
    text = re.sub(r"/\*.*?\*/", "", tp_h.read_text(), flags=re.S)
    declared = set(re.findall(r"\b(qw_tp_[a-z0-9_]+)\s*\(", text))
    assert declared == {"qw_tp_create", "qw_tp_matvec", "qw_tp_local_extent", "qw_tp_free",
                        "qw_tp_exchange_bytes", "qw_tp_arrivals", "qw_tp_bind_peers", "qw_tp_matvec_peer"}
    lib = _native.lib_path().parent / "libqweight_b200_tp.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert declared <= exported
