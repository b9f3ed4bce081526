"""Developer tool: device time of one NAND level (one BR launch + one KS launch) vs level width, CUDA events."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_12761_b200 import _lib as L
from paper_2506_12761_b200 import api as A
from synth import nand_inputs

keys = A.Keys(1005)
srv = A.Server(keys, 0)
widths = [int(x) for x in sys.argv[1:]] or [1, 5, 16, 64, 148, 256, 512, 740, 1024, 1480, 2048, 2960, 4096]
a_bits, b_bits = nand_inputs(max(widths))
a_all = A.to_device(keys.encrypt_bits(a_bits, 7, 0))
b_all = A.to_device(keys.encrypt_bits(b_bits, 7, max(widths)))
for w in widths:
    prog = A.Program.gates(srv, L.NAND, w)
    out = torch.zeros((w, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(a_all[:w], b_all[:w], out)
    torch.cuda.synchronize()
    prog.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    for _ in range(reps):
        prog.eval(a_all[:w], b_all[:w], out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    br_ms, ks_ms, *_ = prog.profile_read()
    print(f"width {w:6d}: {ms:8.2f} ms/level  BR {br_ms / reps:8.2f} ms  KS {ks_ms / reps:7.3f} ms  "
          f"{w / ms * 1e3:9.0f} gates/s", flush=True)
