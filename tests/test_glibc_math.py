"""The device replay of glibc's log / sincos (csrc/glibc_math.cuh), compiled
for the host, is bit-identical to this process's libm -- the functions the
reference's Box-Muller draw calls (rng.hpp:49-62; log -> __log_fma,
sincos -> __sincos_fma on an FMA host).  Random Box-Muller arguments plus
consecutive doubles around every branch boundary.  The device build is
checked through init_states in tests/test_gpu_solver.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cpu_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma " in flags and " avx2 " in flags


@pytest.mark.skipif(not _cpu_has_fma(), reason="libm resolves the non-FMA variants on this CPU")
def test_glibc_math_matches_host_libm(tmp_path):
    exe = tmp_path / "glibc_math_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2605_06921_b200", "csrc"),
                    os.path.join(ROOT, "tests", "glibc_math_check.cpp"), "-o", str(exe), "-lm"],
                   check=True)
    out = subprocess.run([str(exe), "3000000", "20000"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout
