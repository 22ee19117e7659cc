"""Build (CPU) and run (GPU) the C++ drop-in test against include/hmgp/hmgp.hpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_api")


def build_cpp_test():
    lib_dir = os.path.join(ROOT, "paper_2104_07146_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-L", lib_dir, "-lhmgp_cuda",
           f"-Wl,-rpath,{lib_dir}", "-o", EXE]
    subprocess.run(cmd, check=True)


def test_cpp_header_compiles_and_links(hm):
    build_cpp_test()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_api_on_gpu(hm):
    if not os.path.exists(EXE):
        build_cpp_test()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout


def test_cpp_dataset_io(hm):
    """include/hmgp/dataset.hpp (dataset.cpp:46-210): host-only port of test_io.cpp."""
    exe = os.path.join(ROOT, "tests", "cpp", "test_dataset")
    lib_dir = os.path.join(ROOT, "paper_2104_07146_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dataset.cpp"), "-L", lib_dir, "-lhmgp_cuda",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
