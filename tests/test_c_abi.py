"""The C ABI from plain C (no Python binding): tests/c/abi_smoke.c is compiled with gcc against include/vlp.h,
linked to libvlp.so and run (client-side calls only: no GPU needed)."""
import os
import subprocess

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
