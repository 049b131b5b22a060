"""The C++ drop-in (include/btoep_gpu.hpp) compiled like a reference caller,
linked against libbtg.so and run on the GPU (tests/cpp/dropin_example.cpp)."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_cpp_dropin_example_runs(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    exe = tmp_path / "dropin"
    lib_dir = ROOT / "paper_2407_13066_b200"
    r = subprocess.run([gxx, "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/dropin_example.cpp"),
                        f"-L{lib_dir}", "-lbtg", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "OK" in run.stdout
