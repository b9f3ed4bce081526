"""Developer tool: K2F's largest rounding distance |V - round(V)| over whole configurations, measured on the product
kernel with the rounding monitor (vlp_debug_fft_error), plus the decrypted predicate of each run.
    python tools/fft_margin.py [config ...]   (default: 2 3 4)"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import api as A  # noqa: E402
from synth import make_workload  # noqa: E402
from synth.workloads import expected_result  # noqa: E402


def run(cfg):
    wl = make_workload(cfg)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    pk = A.pubkeygen_device(keys, m, wl.key_seed + 1, 0, wl.M)
    db = A.server_encrypt_db_device(m, pk, wl.records, wl.payloads)
    q = A.to_device(keys.encrypt_query(m, wl.query, 7))
    prog = A.Program.velopir(srv, m)
    out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    err = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    A.check(A.lib().vlp_debug_fft_error(ctypes.c_void_p(err.data_ptr())))
    t0 = time.time()
    prog.eval(q, db, out)
    torch.cuda.synchronize()
    A.check(A.lib().vlp_debug_fft_error(None))
    worst = float(np.array([int(err.item())], dtype=np.int64).view(np.float64)[0])
    ok = keys.decrypt_value(A.to_host(out)) == expected_result(wl)
    br = prog.info.br
    print(f"config {cfg} ({wl.name}): {br} BR, {br * 630 * 4096:.3g} limb roundings, largest distance to the "
          f"rounded integer {worst:.3e} (margin 1/2: x{0.5 / worst:.3g}), predicate {'OK' if ok else 'WRONG'}, "
          f"{time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["2", "3", "4"]):
        run(int(c))
