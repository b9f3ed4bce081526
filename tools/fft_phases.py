"""Developer tool: where a K2F step's time goes -- clock64 deltas per phase summed over the warps of one whole
wave, from a dev build with -DVLP_PHASE_TIMING:
    VLP_BUILD_VARIANT=phase VLP_BUILD_DEFS=-DVLP_PHASE_TIMING python -m paper_2506_12761_b200.build
    VLP_LIB=paper_2506_12761_b200/libvlp_phase.so python tools/fft_phases.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402

NAMES = ["digit words (acc reads)", "forward FFT", "key-ring wait", "MAC (TMEM + key LDS)", "TMEM column load",
         "inverse FFT", "round + acc update", "-"]
keys = A.Keys(123)
srv = A.Server(keys, 0)
L.lib().vlp_debug_route(2, 8)
rng = np.random.default_rng(0)
cnt = 8 * torch.cuda.get_device_properties(0).multi_processor_count
x = A.to_device(rng.integers(0, 2 ** 32, (cnt, 632), dtype=np.uint64).astype(np.uint32))
f = L.lib().vlp_debug_phase_read
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 8)()
srv.debug_blind_rotate(x, 630)
f(buf)
srv.debug_blind_rotate(x, 630)
torch.cuda.synchronize()
f(buf)
tot = sum(buf[:7])
per = tot / cnt / 630
print(f"{cnt} bootstraps x 630 steps: {per:.0f} warp-cycles per step (SM clock)")
for k in range(7):
    print(f"  {NAMES[k]:28s} {buf[k] / tot * 100:5.1f} %  {buf[k] / cnt / 630:8.0f} cycles/step")

# per-CTA spread of one wave (globaltimer at CTA start / end, SM id)
g = L.lib().vlp_debug_cta_read
g.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
cb = (ctypes.c_ulonglong * (11 * 1024))()
g(cb)
srv.debug_blind_rotate(x, 630)
torch.cuda.synchronize()
g(cb)
sm = torch.cuda.get_device_properties(0).multi_processor_count
st = np.array([cb[3 * i] for i in range(sm)], dtype=np.float64)
en = np.array([cb[3 * i + 1] for i in range(sm)], dtype=np.float64)
ids = np.array([cb[3 * i + 2] for i in range(sm)])
dur = (en - st) / 1e6
t0 = st.min()
print(f"per-CTA duration ms: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f}; "
      f"start spread {(st.max() - t0) / 1e3:.1f} us; end spread {(en.max() - en.min()) / 1e6:.2f} ms; "
      f"wave {(en.max() - t0) / 1e6:.2f} ms")
order = np.argsort(dur)
print("fastest SMs", [(int(ids[i]), round(float(dur[i]), 2)) for i in order[:6]])
print("slowest SMs", [(int(ids[i]), round(float(dur[i]), 2)) for i in order[-6:]])
ph = np.array([[cb[3 * 1024 + 8 * i + k] for k in range(7)] for i in range(sm)], dtype=np.float64) / (8 * 630)
for name, sel in (("fastest", order[:6]), ("slowest", order[-6:])):
    m = ph[sel].mean(axis=0)
    print(f"{name} CTAs, cycles per warp-step by phase: " + ", ".join(f"{NAMES[k].split()[0]} {m[k]:.0f}" for k in range(7)))
