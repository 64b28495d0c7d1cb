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
