"""The C++ drop-in headers (include/lorakv/*.hpp, same operator API as the reference's
proj/include/lorakv) and their C++ parity suites (tests/cpp/*.cpp, modelled on the reference's
tests/test_attention.cpp, test_kvcache.cpp and test_lora.cpp).

CPU: the headers compile as C++20 and C++17 and the suite links against liblorakv_b200.so.
GPU: the suite runs on the B200 -- every operator goes through the C ABI to the CUDA kernels and is
compared with the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BIN = os.path.join(CPP, "build", "lorakv_cpp_tests")


def build():
    from oracle import checker
    from paper_2602_01053_b200 import abi
    checker.build_oracle()
    if not os.path.exists(abi.lib_path()):
        abi.build()
    res = subprocess.run(["make", "-C", CPP, "-j8"], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]


def test_headers_compile_and_suite_links():
    build()
    assert os.path.exists(BIN)
    probe = ('#include "lorakv/attention.hpp"\n#include "lorakv/kvcache.hpp"\n#include "lorakv/lora.hpp"\n'
             '#include "lorakv/device.hpp"\n#include "lorakv/replay.hpp"\n#include "lorakv/fuzz.hpp"\nint main() { return 0; }\n')
    for std in ("c++17", "c++20"):
        res = subprocess.run(["g++", f"-std={std}", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                              "-I" + os.path.join(ROOT, "include"), "-x", "c++", "-"],
                             input=probe, capture_output=True, text=True)
        assert res.returncode == 0, res.stderr[-3000:]


def test_headers_fail_loudly_without_a_gpu():
    """No CPU fallback behind the headers: without a CUDA device the first operator throws."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    build()
    res = subprocess.run([BIN, "closed-form MAC counts"], capture_output=True, text=True)   # host-only integer case
    assert res.returncode == 0, res.stdout + res.stderr
    res = subprocess.run([BIN, "single cached token"], capture_output=True, text=True)
    assert res.returncode != 0
    assert "needs a CUDA device" in res.stderr or "CUDA" in res.stderr


@pytest.mark.gpu
def test_cpp_parity_suite_on_gpu():
    build()
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    tail = (res.stdout + res.stderr)[-6000:]
    assert res.returncode == 0, tail
    assert "failed: 0 | assertions" in res.stdout, tail
