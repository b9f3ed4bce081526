"""Developer tool: K2F time per wave against the number of waves in one level (persistent CTAs drift apart over
many waves; VLP_FFT_WAVES=k splits a level into launches of at most k waves).
    [VLP_FFT_WAVES=k] python tools/wave_drift.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402

keys = A.Keys(123)
srv = A.Server(keys, 0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
rng = np.random.default_rng(0)
assert L.lib().vlp_debug_route(2, 8) == 0
for waves in [int(x) for x in (sys.argv[1:] or ["1", "8", "64", "221"])]:
    cnt = 8 * sms * waves
    x = A.to_device(rng.integers(0, 2 ** 32, (cnt, 632), dtype=np.uint64).astype(np.uint32))
    srv.debug_blind_rotate(x, 630)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    srv.debug_blind_rotate(x, 630)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"VLP_FFT_WAVES={os.environ.get('VLP_FFT_WAVES', '-')}: {waves} waves, {ms / waves:.2f} ms per wave, "
          f"{cnt / ms * 1e3:.0f} BR/s", flush=True)
    del x
    torch.cuda.empty_cache()
