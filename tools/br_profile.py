"""Developer tool: one blind-rotation level (630 steps) on a chosen engine, for ncu captures.
    python tools/br_profile.py ENGINE PARAM COUNT   (ENGINE 1 = NTT (PARAM = VLP_BR_BOOT meaning), 2 = K2F (PARAM warps))"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402

eng, par, cnt = (int(x) for x in sys.argv[1:4])
keys = A.Keys(123)
srv = A.Server(keys, 0)
assert L.lib().vlp_debug_route(eng, par) == 0
rng = np.random.default_rng(0)
x = A.to_device(rng.integers(0, 2 ** 32, (cnt, 632), dtype=np.uint64).astype(np.uint32))
srv.debug_blind_rotate(x, 630)
torch.cuda.synchronize()
print("done", flush=True)
