"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares; the product path fails loudly without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rsvd_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsvd_b200_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header():
    from paper_2110_03423_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.EXPORTS) == names
    assert b"sm_100a" in lib.rsvd_b200_version()


def test_library_is_sm100a():
    from paper_2110_03423_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_kernels_use_tma_and_dmma():
    from paper_2110_03423_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True,
                          timeout=600).stdout
    assert "DMMA" in sass  # FP64 tensor-core MMA
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "UTCHMMA" in sass  # tcgen05.mma (the FP32 path's 3xTF32 products)
    assert "LDTM" in sass  # tcgen05.ld: accumulators read back from TMEM


def test_sketch_width_matches_reference_rule():
    from paper_2110_03423_b200 import _lib
    import ctypes as C
    lib = _lib.load()
    cfg = _lib.Config()
    lib.rsvd_b200_config_default(C.byref(cfg))
    assert (cfg.k, cfg.oversample, cfg.power_q, cfg.seed, cfg.epsilon, cfg.epsilon_mode) == \
        (1, 10, 2, 0, 0.5, 0)
    cfg.k = 5
    cfg.epsilon = 0.25
    cfg.epsilon_mode = 1
    assert lib.rsvd_b200_sketch_width(C.byref(cfg), 100, 80) == 20  # test_rsvd.cpp:224-234
    cfg.epsilon = 0.01
    assert lib.rsvd_b200_sketch_width(C.byref(cfg), 100, 80) == 80
    cfg.epsilon_mode = 0
    assert lib.rsvd_b200_sketch_width(C.byref(cfg), 100, 80) == 15


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2110_03423_b200 as P
    with pytest.raises(P.DeviceError):
        P.Solver(0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2110_03423_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.lower().replace("oracles", ""), f
