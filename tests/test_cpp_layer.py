"""The C++ host layer (include/questkv_b200.hpp): compiled with g++ -std=c++20 against the
in-tree libquestkv_b200.so and the C oracle (test infrastructure), then run.

CPU: host-side checks and "no device -> std::runtime_error" (no CPU fallback).
GPU: the reference's known-answer cases restated in C++ plus random parity against the
oracle (metadata, scores and pages bitwise; outputs rel-L2 <= 1e-5)."""

import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
LIB_DIR = os.path.join(ROOT, "paper_2406_10774_b200")
ORACLE_DIR = os.path.join(ROOT, "oracle")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    if not os.path.exists(os.path.join(LIB_DIR, "libquestkv_b200.so")):
        pytest.fail("libquestkv_b200.so missing: run __graft_entry__.build()")
    if not os.path.exists(os.path.join(ORACLE_DIR, "liboracle.so")):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "oracle"], check=True)
    out = str(tmp_path_factory.mktemp("cpp") / "test_questkv_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", ORACLE_DIR,
           os.path.join(ROOT, "tests", "cpp", "test_questkv_b200.cpp"), "-o", out,
           "-L", LIB_DIR, "-lquestkv_b200", "-L", ORACLE_DIR, "-loracle",
           f"-Wl,-rpath,{LIB_DIR}", f"-Wl,-rpath,{ORACLE_DIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return out


def test_cpp_layer_host_checks(binary):
    r = subprocess.run([binary, "--cpu"], capture_output=True, text=True, timeout=120,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_layer_parity(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


REF_DIR = os.path.join(ORACLE_DIR, "_ref")
COMPAT_REF = os.path.join(REF_DIR, "compat_check_ref")
COMPAT_B200 = os.path.join(REF_DIR, "compat_check_b200")


def test_reference_callers_compile_unchanged_against_compat_headers():
    """R/core/src/metrics.cpp and policies.cpp (the reference's own callers of the operator
    API) compile and link UNCHANGED against include/questkv_compat (questkv:: bound to the
    B200 library).  Built by oracle/Makefile `compat` from the read-only sources when
    /root/reference exists; the GPU box receives the prebuilt binaries."""
    if os.path.isdir("/root/reference/proj/core/src"):
        r = subprocess.run(["make", "-s", "-C", ORACLE_DIR, "compat"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
    if not os.path.exists(COMPAT_B200):
        pytest.skip("compat checks not built (needs /root/reference)")
    assert os.path.exists(COMPAT_REF)


@pytest.mark.gpu
def test_reference_callers_on_the_gpu_match_the_reference():
    """The same driver (reference API only) against the unmodified reference and against
    metrics.cpp/policies.cpp running on the GPU library: selections (page-ordered and
    arbitrary PageScore vectors), logits, scores, recall, byte tallies, oracle sparsity and
    every policy's token set equal; outputs within 1e-5 relative L2; softmax weights and
    accumulated H2O mass within 1e-12; weights_sum_check within 1e-6 of the reference's."""
    import json

    import numpy as np

    if not (os.path.exists(COMPAT_REF) and os.path.exists(COMPAT_B200)):
        pytest.fail("oracle/_ref compat checks missing (build them where /root/reference exists)")
    ref = json.loads(subprocess.run([COMPAT_REF], capture_output=True, text=True, timeout=300,
                                    check=True).stdout)
    got = json.loads(subprocess.run([COMPAT_B200], capture_output=True, text=True, timeout=300,
                                    check=True).stdout)
    assert ref.keys() == got.keys()
    exact = ["scores", "pages", "pages_shuffled", "pages_shuffled_noforce", "pages_few",
             "pages_few_all", "logits_all", "logits_sub", "recall", "bytes", "fraction_model",
             "oracle_sparsity", "policy_full", "policy_quest", "policy_h2o", "policy_tova",
             "policy_streaming"]
    for k in exact:
        assert got[k] == ref[k], k
    for k in ("sparse", "full", "tokens"):
        a, b = np.array(got[k]), np.array(ref[k])
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5, k
    for k in ("softmax_sub", "h2o_scores"):
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-12, atol=1e-15, err_msg=k)
    for k in ("sparse_wsum", "full_wsum", "tokens_wsum"):
        assert abs(got[k][0] - ref[k][0]) <= 1e-6, k
    assert abs(got["output_error"][0] - ref["output_error"][0]) <= 1e-5
