"""CPU suite: the C-ABI library loads and exports every declared symbol; the
product never depends on the oracle; no-GPU behaviour fails loudly."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_11645_b200", "librstg.so")
HOSTLIB = os.path.join(ROOT, "paper_2603_11645_b200", "librst_b200.so")


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rstg.h")).read()
    return sorted(set(re.findall(r"\b(rstg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_symbols():
    syms = declared_symbols()
    assert "rstg_run" in syms and "rstg_graph_create" in syms and len(syms) >= 15


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("librstg.so not built")
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in include/rstg.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_python_binding_lists_exports():
    import paper_2603_11645_b200 as P

    assert set(P.EXPORTS) == set(declared_symbols())


def test_sm100a_code_in_library():
    if not os.path.exists(LIB):
        pytest.skip("librstg.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_11645_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "rst_oracle" not in text, f
                assert "librst_ref" not in text, f


def test_no_gpu_fails_loudly():
    """Without a device the library reports an error instead of computing
    anything on the CPU."""
    import paper_2603_11645_b200 as P

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.CudaError):
        P.DeviceGraph.generate("path:4")


def test_host_mirror_exports():
    if not os.path.exists(HOSTLIB):
        pytest.skip("librst_b200.so not built")
    out = subprocess.run(["nm", "-DC", "--defined-only", HOSTLIB], capture_output=True,
                         text=True).stdout
    for sym in ("rst::run_algorithm", "rst::cc_euler_rst", "rst::pr_rst", "rst::bfs_rst",
                "rst::cc_spanning_forest", "rst::euler_root_forest", "rst::build_csr",
                "rst::validate_rooted_forest", "rst::bench_row"):
        assert sym in out, sym
