"""The device generator's restatement of glibc 2.39's FMA-path log and sincos
(paper_2110_03423_b200/csrc/glibc_libm.cuh) against this host's libm, bit for bit.

The same header is compiled for the host here (every step an explicit single rounding,
so host and device evaluate the identical operation sequence) and checked on the inputs
the reference sampler feeds libm (rng.cpp:36-44) plus arbitrary arguments across every
branch. The GPU side is pinned by tests/test_gpu_parity.py::test_device_normals_vs_reference.
"""
import os
import subprocess

import pytest

from conftest import ROOT


def _cpu_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma " in flags and " avx2 " in flags


@pytest.mark.skipif(not _cpu_has_fma(), reason="glibc selects its FMA builds only on AVX2+FMA hosts")
def test_restated_libm_bit_exact(tmp_path):
    exe = str(tmp_path / "glibc_libm_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", exe,
                    os.path.join(ROOT, "tests", "glibc_libm_check.cpp"), "-lm"], check=True)
    r = subprocess.run([exe, "3000000", "42"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
    assert r.stdout.strip().endswith("of 15000000")


def test_tables_match_this_libm():
    """csrc/glibc239_tables.h is what tools/gen_glibc_tables.py extracts from this libm."""
    import hashlib
    hdr = open(os.path.join(ROOT, "paper_2110_03423_b200", "csrc", "glibc239_tables.h")).read()
    blob = open("/lib/x86_64-linux-gnu/libm.so.6", "rb").read()
    assert f"sha256 {hashlib.sha256(blob).hexdigest()[:16]}" in hdr
