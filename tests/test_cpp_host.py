"""The C++ host API (include/absim_b200.hpp) over the C ABI: compiles on the
CPU; on a B200 it re-runs the reference's known-answer tests
(tests/cpp/host_known_answers.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "host_known_answers.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "host_known_answers")
LIBDIR = os.path.join(ROOT, "paper_2301_06984_b200", "_lib")


def _compile():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", f"-I{ROOT}/include", SRC, f"-L{LIBDIR}",
                    "-labsim_gpu", f"-Wl,-rpath,{LIBDIR}", "-o", OUT], check=True)


def test_cpp_host_compiles(engine):
    _compile()
    assert os.path.exists(OUT)


@pytest.mark.gpu
def test_cpp_host_known_answers(engine):
    _compile()
    r = subprocess.run([OUT], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
