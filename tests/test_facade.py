"""The header-only C++ facade (damf_engine.hpp) compiles against the C ABI
and, on a GPU, reproduces a reference known answer through it, and runs the
reference's three constructors (engine.hpp:29-34), accessors and DAMF v1
persistence."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "build", "facade_example")


def build():
    lib = os.path.join(ROOT, "paper_2306_08967_b200")
    subprocess.run(["g++", "-std=c++17", "-O2", "-o", EXE,
                    os.path.join(ROOT, "tests", "facade_example.cpp"),
                    f"-L{lib}", "-ldamf_gpu", f"-Wl,-rpath,{lib}"], check=True)


def test_facade_compiles_and_links():
    build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_facade_known_answer_on_gpu(tmp_path):
    build()
    r = subprocess.run([EXE, str(tmp_path / "facade.damf")], capture_output=True, text=True,
                       timeout=120)
    print(r.stdout)
    assert r.returncode == 0 and "facade ok" in r.stdout
