"""The drop-in C++ API: the reference's unit-test cases compiled against
paper_2605_06921_b200/cpp/include/mqo/*.hpp and run on the B200
(cpp/tests/facade_tests.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("devices", [None, "0,0"])
def test_facade_cpp_suite(cuda_ok, devices):
    """devices "0,0": every solve_pooled of the re-hosted suite runs sharded
    over two ranks (MQO_DEVICES -> mqo_solve_devices, in-process exchange on
    one GPU) and must give the same answers (test_solver.cpp:221-233)."""
    pkg = os.path.join(ROOT, "paper_2605_06921_b200")
    exe = os.path.join(pkg, "cpp", "tests", "facade_tests.bin")
    if not os.path.exists(exe):  # compile against the shipped .so files
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(pkg, "cpp", "include"),
                        "-I", os.path.join(ROOT, "include"), "-o", exe,
                        os.path.join(pkg, "cpp", "tests", "facade_tests.cpp"), f"-L{pkg}",
                        "-lmqo_core_b200", "-lmqo_b200", f"-Wl,-rpath,{pkg}"], check=True)
    env = dict(os.environ)
    if devices:
        env["MQO_DEVICES"] = devices
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
