"""The C ABI from plain C (no Python binding): tests/c/abi_smoke.c is compiled with gcc against include/vlp.h,
linked to libvlp.so and run (client-side calls, no GPU); tests/c/abi_server.c runs the server calls on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_uses_the_abi(tmp_path):
    from paper_2506_12761_b200 import build as B
    lib = B.LIB
    exe = tmp_path / "abi_smoke"
    subprocess.check_call(["gcc", "-std=c99", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c", "abi_smoke.c"), lib, "-o", str(exe),
                           f"-Wl,-rpath,{os.path.dirname(lib)}"])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "c abi ok" in r.stdout


@pytest.mark.gpu
def test_c_program_runs_the_server_calls(tmp_path):
    """tests/c/abi_server.c: vlp_server_create, vlp_gate_batch, vlp_server_eval (two shards and all records) and
    vlp_server_combine from plain C with CUDA-runtime device buffers; sharded + combine is byte-identical to the
    single evaluation (R15) and decrypts to the plain predicate."""
    from paper_2506_12761_b200 import build as B
    lib = B.LIB
    exe = tmp_path / "abi_server"
    subprocess.check_call(["gcc", "-std=c99", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "c", "abi_server.c"), lib, "-o", str(exe),
                           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.dirname(lib)}",
                           "-Wl,-rpath,/usr/local/cuda/lib64"])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "c abi server ok" in r.stdout


def test_c_server_program_compiles(tmp_path):
    """The GPU-side C user above also compiles and links on a box without a GPU (header / symbol check)."""
    from paper_2506_12761_b200 import build as B
    lib = B.LIB
    subprocess.check_call(["gcc", "-std=c99", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "c", "abi_server.c"), lib, "-o", str(tmp_path / "abi_server"),
                           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{os.path.dirname(lib)}"])
