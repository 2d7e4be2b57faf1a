"""The drop-in claim, checked with the reference's own code: its test files and its only production callers (step() in
engine.hpp:279, run_trace() in trace.hpp:85) are compiled from where they lie against THIS repository's headers
(include/lorakv comes first on the include path; engine.hpp / trace.hpp, which have no counterpart here, come from the
reference) and -- on the GPU box -- run, linked with liblorakv_b200.so (oracle/Makefile `ref_tests` ->
oracle/_ref/ref_tests_on_b200).  doctest is not vendored in the reference tree; tests/cpp/shim/doctest.h stands in.

CPU (here, where /root/reference exists): every file passes `g++ -fsyntax-only`, and step<float> / step<double> / run_trace
instantiate.  GPU: the binary built here runs all 81 cases of test_attention / test_kvcache / test_lora / test_matrix /
test_engine / test_trace with zero failures."""
import os
import subprocess
import sysconfig

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
JSON_INC = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann")
INCLUDES = ["-I" + os.path.join(ROOT, "tests", "cpp", "shim"), "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(REF, "include"),
            "-I" + JSON_INC]
FILES = ["test_attention.cpp", "test_lora.cpp", "test_kvcache.cpp", "test_matrix.cpp", "test_engine.cpp", "test_trace.cpp"]

needs_reference = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")), reason="/root/reference is not present on this box")


@needs_reference
@pytest.mark.parametrize("name", FILES)
def test_reference_test_file_compiles_against_the_dropin_headers(name):
    res = subprocess.run(["g++", "-std=c++20", "-fsyntax-only"] + INCLUDES + [os.path.join(REF, "tests", name)],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-3000:]


@needs_reference
def test_step_and_run_trace_instantiate_for_float_and_double():
    """engine.hpp step<T> is the only production caller of gqa_attention and of KvStore::append_* (SURVEY 1); trace.hpp
    run_trace<T> drives it.  Explicit instantiation compiles every member they touch: hidden_rows / append_hidden /
    recompute_overwrite, dtype_name<T>, the views, bytes(), tokens()."""
    tu = ('#include "lorakv/trace.hpp"\n'
          "namespace lorakv {\n"
          "template StepOutput<float> step<float>(const Model<float>&, KvStore<float>&, idx, const std::vector<std::int32_t>&, StepMode,\n"
          "                                        const BlockConfig&, FlopCounter&, StepCapture<float>*);\n"
          "template StepOutput<double> step<double>(const Model<double>&, KvStore<double>&, idx, const std::vector<std::int32_t>&, StepMode,\n"
          "                                          const BlockConfig&, FlopCounter&, StepCapture<double>*);\n"
          "}\n"
          "int main() { lorakv::KvStore<float> a(lorakv::CacheScheme{}, lorakv::StoreDims{1, 4, 4, 0, 1}); lorakv::KvStore<float> b = a;\n"
          "             return a == b ? 0 : 1; }\n")
    res = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-"] + INCLUDES, input=tu, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-3000:]


@needs_reference
def test_the_suite_binary_builds_here():
    from oracle import checker
    from paper_2602_01053_b200 import abi
    if not os.path.exists(abi.lib_path()):
        abi.build()
    path = checker.build_ref_tests()
    assert path and os.path.exists(path)


@pytest.mark.gpu
def test_reference_suites_pass_on_the_b200_path():
    """Runs the binary built in the dev container (it travels with the snapshot like every other built file)."""
    from oracle import checker
    if not os.path.exists(checker.REF_TESTS):
        pytest.skip("oracle/_ref/ref_tests_on_b200 was not built (no /root/reference where the tree was built)")
    res = subprocess.run([checker.REF_TESTS], capture_output=True, text=True, timeout=900)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    summary = [ln for ln in res.stdout.splitlines() if ln.startswith("[doctest-shim]")]
    assert summary and "| failed: 0 |" in summary[0] and summary[0].rstrip().endswith("failed: 0"), tail
    n_cases = int(summary[0].split("test cases:")[1].split("|")[0])
    assert n_cases >= 81, summary[0]          # 16 + 15 + 9 + 10 + 17 + 14 cases of the six files
