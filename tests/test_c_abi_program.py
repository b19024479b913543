"""A plain C program compiled against include/cfr_b200.h (examples/kuhn_c_abi.c):
the header is usable from C as declared, and the library links without Python.
Host half (game creation, Table 7 dimensions, qbase, canonical order) on CPU;
the solver half (1000 vanilla CFR iterations, Kuhn value -1/18) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2408_14778_b200")


@pytest.fixture(scope="module")
def kuhn_exe(tmp_path_factory):
    import paper_2408_14778_b200 as pb

    pb.build()
    exe = str(tmp_path_factory.mktemp("cabi") / "kuhn_c_abi")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "kuhn_c_abi.c"),
                           "-L", LIBDIR, "-lcfr_b200", f"-Wl,-rpath,{LIBDIR}", "-L", "/usr/local/cuda/lib64",
                           "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm", "-o", exe])
    return exe


def test_c_program_host_half(kuhn_exe):
    out = subprocess.run([kuhn_exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "V=58 terminals=30" in out.stdout and "host half ok" in out.stdout


@pytest.mark.gpu
def test_c_program_gpu_half(kuhn_exe, cuda):
    out = subprocess.run([kuhn_exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu half ok" in out.stdout
