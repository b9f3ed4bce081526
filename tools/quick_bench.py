"""Developer tool: time the NAND gate batch (BR + KS kernels) and config 2 on one GPU with CUDA events."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import numpy as np
import torch

from paper_2506_12761_b200 import _lib as L
from paper_2506_12761_b200 import api as A
from synth import make_workload, nand_inputs


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14
    t0 = time.time()
    keys = A.Keys(1005)
    srv = A.Server(keys, 0)
    print(f"keygen+server {time.time() - t0:.1f}s", flush=True)
    a_bits, b_bits = nand_inputs(count)
    a = A.to_device(keys.encrypt_bits(a_bits, 2005, 0))
    b = A.to_device(keys.encrypt_bits(b_bits, 2005, count))
    prog = A.Program.gates(srv, L.NAND, count)
    out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(a, b, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 2
    for _ in range(reps):
        prog.eval(a, b, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ok = np.array_equal(keys.decrypt_bits(A.to_host(out)), 1 - (a_bits & b_bits))
    print(f"NAND x{count}: {ms:.1f} ms -> {count / ms * 1e3:.0f} gates/s  correct={ok}", flush=True)
    if len(sys.argv) > 2:
        wl = make_workload(2)
        m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
        q = A.to_device(keys.encrypt_query(m, wl.query, 7))
        db = A.to_device(keys.encrypt_db(m, wl.records, wl.payloads, 9))
        p2 = A.Program.velopir(srv, m)
        o2 = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        p2.eval(q, db, o2)
        torch.cuda.synchronize()
        e0.record()
        p2.eval(q, db, o2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"config2: {ms:.1f} ms, {p2.info.br / ms * 1e3:.0f} BR/s, {wl.M / ms * 1e3:.1f} records/s, "
              f"result {keys.decrypt_value(A.to_host(o2))}", flush=True)


if __name__ == "__main__":
    main()
