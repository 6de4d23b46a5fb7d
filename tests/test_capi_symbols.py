"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every function declared in include/xigemm_c.h; the Python mirror
binds exactly those; calling compute without a device fails loudly."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "xigemm_c.h")
LIB = os.path.join(ROOT, "paper_2403_06924_b200", "lib", "libxigemm_b200.so")


def declared():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    assert all(re.search(rf"\bT {n}$", out, re.M) for n in names)


def test_python_binding_covers_header():
    from paper_2403_06924_b200 import _lib
    assert set(_lib.exported_symbols()) == set(declared())


def test_cpp_dropin_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    for sym in ["xigemm::xigemm(xigemm::DenseMatrix const&, xigemm::DenseMatrix const&, xigemm::XigemmConfig const&)",
                "xigemm::quantize(", "xigemm::gemm_int(", "xigemm::spmm_int(", "xigemm::reduce_a(",
                "xigemm::quantize_csr(", "xigemm::dequant_product(", "xigemm::get_avg_vectors(",
                "xigemm::quantized_gemm_full_residual(", "xigemm::csr_transpose<signed char>"]:
        assert sym in out, sym


def test_config_default_and_limits():
    from paper_2403_06924_b200 import _lib
    lib = _lib.lib()
    lib.xg_config_default.restype = _lib.XgConfig
    c = lib.xg_config_default()
    assert (c.bits, c.threshold, c.density_limit, c.scheme, c.policy, c.rounding) == (8, 0.5, 0.3, 0, 1, 1)
    assert lib.xg_gemm_max_inner(8) == 16384 and lib.xg_gemm_max_inner(4) == 1 << 22


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2403_06924_b200 import _lib
    assert _lib.lib().xg_device_ok() == 0
    import numpy as np
    import paper_2403_06924_b200 as xg
    with pytest.raises(Exception):
        xg.xigemm_host(np.ones((4, 4), np.float32), np.ones((4, 4), np.float32))


def test_shard_api_validation_without_device():
    """xg_shard_create rejects bad layouts with XG_EINVAL (the reference's
    std::invalid_argument class) before touching the device."""
    import ctypes as C
    from paper_2403_06924_b200 import _lib
    lib = _lib.lib()
    cfg = _lib.XgConfig(8, 0.5, 0.3, 1, 0, 1)
    h = C.c_void_p()
    buf = (C.c_float * 16)()
    rows = (C.c_int * 2)(4, 4)

    def create(rank, nranks, rr, k, n, cfg_=cfg, a=buf, out=buf):
        return lib.xg_shard_create(a, buf, None, 1.0, 0.0, rank, nranks, rr, k, n, C.byref(cfg_), 1, out,
                                   C.byref(h))

    assert create(2, 2, rows, 4, 4) == 1                         # rank out of range
    assert create(0, 2, (C.c_int * 2)(4, 0), 4, 4) == 1          # empty shard
    assert create(0, 2, rows, 16385, 4) == 1                     # int8 K limit (quantize.cpp:197-200)
    assert create(0, 2, rows, 4, 4, a=None) == 1                 # null matrix
    bad = _lib.XgConfig(8, 0.5, 1.5, 1, 0, 1)
    assert create(0, 2, rows, 4, 4, cfg_=bad) == 1               # s outside (0, 1] (pipeline.cpp:153-160)
    assert b"density limit" in lib.xg_last_error()
    assert lib.xg_shard_step(None, 0, None) == 1
