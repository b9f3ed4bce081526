"""Developer tool: quick GPU check of the K2F (FP64 FFT) blind-rotation engine against the oracle, and a
level-time comparison of the engines.  Not a test (tests/test_gpu_parity.py holds those).

    python tools/fft_check.py [--time]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402


def main():
    keys = A.Keys(123)
    srv = A.Server(keys, 0)
    ok = O.OracleKeys(123)
    rng = np.random.default_rng(1)
    cts = rng.integers(0, 2 ** 32, (9, 632), dtype=np.uint64).astype(np.uint32)
    cts[:, 631] = 0
    cts[4, :630] = 0
    dev = A.to_device(cts)
    for W in (1, 3, 8):
        assert L.lib().vlp_debug_route(2, W) == 0
        for steps in (1, 2, 7):
            got = A.to_host(srv.debug_blind_rotate(dev, steps))
            bad = 0
            for i in range(9):
                want = ok.blind_rotate(cts[i, :631], steps)
                if not np.array_equal(got[i], want):
                    bad += 1
                    d = np.flatnonzero(got[i] != want)
                    print(f"W={W} steps={steps} row {i}: {len(d)} words differ, first {d[:6]}, "
                          f"got {got[i][d[:3]]} want {want[d[:3]]}", flush=True)
            print(f"W={W} steps={steps}: {9 - bad}/9 rows byte-equal", flush=True)
    L.lib().vlp_debug_route(0, 0)
    if "--time" in sys.argv:
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        for name, eng, par, cnt in (("ntt K2 5/SM", 1, 5, 5 * sms), ("fft K2F 8/SM", 2, 8, 8 * sms),
                                    ("fft K2F 8/SM x4", 2, 8, 32 * sms)):
            assert L.lib().vlp_debug_route(eng, par) == 0
            x = A.to_device(rng.integers(0, 2 ** 32, (cnt, 632), dtype=np.uint64).astype(np.uint32))
            srv.debug_blind_rotate(x, 630)
            torch.cuda.synchronize()
            t0 = time.time()
            srv.debug_blind_rotate(x, 630)
            torch.cuda.synchronize()
            dt = time.time() - t0
            print(f"{name}: {cnt} BR x 630 steps in {dt * 1e3:.1f} ms -> {cnt / dt:.0f} BR/s", flush=True)
        L.lib().vlp_debug_route(0, 0)


if __name__ == "__main__":
    main()
