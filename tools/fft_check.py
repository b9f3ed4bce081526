"""Developer tool: quick GPU check of the K2F (FP64 FFT) blind-rotation engine against the NTT engine (both in
libvlp; the oracle parity tests are in tests/test_gpu_parity.py), and a level-time comparison of the engines.

    python tools/fft_check.py [--time]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402


def main():
    keys = A.Keys(123)
    srv = A.Server(keys, 0)
    rng = np.random.default_rng(1)
    cts = rng.integers(0, 2 ** 32, (9, 632), dtype=np.uint64).astype(np.uint32)
    cts[:, 631] = 0
    cts[4, :630] = 0
    dev = A.to_device(cts)
    for steps in (1, 2, 7):
        assert L.lib().vlp_debug_route(1, 5) == 0  # the NTT engine's bytes as the reference
        ref = A.to_host(srv.debug_blind_rotate(dev, steps))
        for W in (1, 3, 8):
            assert L.lib().vlp_debug_route(2, W) == 0
            got = A.to_host(srv.debug_blind_rotate(dev, steps))
            bad = [i for i in range(9) if not np.array_equal(got[i], ref[i])]
            for i in bad[:3]:
                d = np.flatnonzero(got[i] != ref[i])
                print(f"W={W} steps={steps} row {i}: {len(d)} words differ from the NTT engine, first {d[:6]}", flush=True)
            print(f"W={W} steps={steps}: {9 - len(bad)}/9 rows byte-equal to the NTT engine", flush=True)
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
