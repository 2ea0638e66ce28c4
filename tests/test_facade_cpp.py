"""Compiles tests/cpp/facade_test.cpp (the reference's test_engine.cpp cases
written against include/econosim_b200.hpp) and runs it: on CPU against the
host build of the engine source, on the GPU against the sm_100a library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_and_run(lib_dir, lib_name, tmp_path):
    exe = str(tmp_path / "facade_test")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), "-L" + lib_dir,
                    "-l:" + lib_name, "-Wl,-rpath," + lib_dir, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all facade checks passed" in r.stdout


def test_facade_on_host_build(tmp_path):
    build_and_run(os.path.join(ROOT, "tests", "_hostsim"), "libeconoserve_hostsim.so", tmp_path)


@pytest.mark.gpu
def test_facade_on_device(tmp_path):
    build_and_run(os.path.join(ROOT, "paper_2411_06364_b200", "_lib"), "libeconoserve_b200.so", tmp_path)
