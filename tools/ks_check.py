"""Developer tool: the time of 2048- and 16384-wide K3T (tcgen05 int8 key switch) launches through the debug call
(CUDA events), and with --level the key-switch time inside a NAND program.  The oracle parity tests of K3T live in
tests/test_gpu_parity.py.
    python tools/ks_check.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import api as A  # noqa: E402


def main():
    keys = A.Keys(123)
    srv = A.Server(keys, 0)
    rng = np.random.default_rng(3)
    for count in (2048, 16384):
        nl = A.to_device(rng.integers(0, 2 ** 32, (count, 1028), dtype=np.uint64).astype(np.uint32))
        srv.debug_keyswitch(nl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            srv.debug_keyswitch(nl)
        e1.record()
        torch.cuda.synchronize()
        print(f"{count} key switches: {e0.elapsed_time(e1) / 5:.3f} ms per level (incl. debug-call overheads)", flush=True)


if __name__ == "__main__" and (len(sys.argv) == 1 or sys.argv[1] != "--level"):
    main()


def level_time(count=2048, reps=5):
    """CUDA-event time of the key-switch launches (prologue + GEMM) of one `count`-wide level: a NAND gate
    program (one BR level + one KS level), profiled by the library (vlp_program_profile)."""
    from paper_2506_12761_b200 import _lib as L
    keys = A.Keys(123)
    srv = A.Server(keys, 0)
    rng = np.random.default_rng(5)
    a = A.to_device(keys.encrypt_bits(rng.integers(0, 2, count, dtype=np.uint8), 1, 0))
    b = A.to_device(keys.encrypt_bits(rng.integers(0, 2, count, dtype=np.uint8), 1, count))
    prog = A.Program.gates(srv, L.NAND, count)
    out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(a, b, out)
    prog.profile(True)
    for _ in range(reps):
        prog.eval(a, b, out)
    torch.cuda.synchronize()
    br_ms, ks_ms, nb, nk = prog.profile_read()
    print(f"{count}-wide level: key switch {ks_ms / reps * 1e3:.1f} us (CUDA events), blind rotation {br_ms / reps:.2f} ms",
          flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--level":
    for c in (2048, 16384):
        level_time(c)
