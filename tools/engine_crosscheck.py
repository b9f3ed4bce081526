"""Developer tool (GPU): every gate output of whole configurations computed twice, by the default routing (K2F FP64-FFT
waves + tails) and by the integer-NTT engine alone (vlp_debug_route(1, 5)), with VLP_F_KEEP_ALL so each intermediate
keeps its own scratch row; the two exact engines share no arithmetic, so byte equality of
every row is a full-size cross-check of both.  Also checks the decrypted predicate.
    python tools/engine_crosscheck.py [config ...]   (default: 2 3)"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402
from synth import make_workload  # noqa: E402
from synth.workloads import expected_result  # noqa: E402


def run(cfg):
    wl = make_workload(cfg)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags | L.F_KEEP_ALL)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    pk = A.pubkeygen_device(keys, m, wl.key_seed + 1, 0, wl.M)
    db = A.server_encrypt_db_device(m, pk, wl.records, wl.payloads)
    q = A.to_device(keys.encrypt_query(m, wl.query, 7))
    prog = A.Program.velopir(srv, m)
    outs, rows = [], []
    for name, route in (("default (K2F waves + tails)", (0, 0)), ("NTT engine only", (1, 5))):
        A.check(L.lib().vlp_debug_route(*route))
        out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        prog.scratch.zero_()
        torch.cuda.synchronize()
        t0 = time.time()
        prog.eval(q, db, out)
        torch.cuda.synchronize()
        dt = time.time() - t0
        ok = keys.decrypt_value(A.to_host(out)) == expected_result(wl)
        print(f"config {cfg} ({wl.name}) {name}: {prog.info.br} BR in {dt:.2f} s, predicate {'OK' if ok else 'WRONG'}",
              flush=True)
        outs.append(out)
        rows.append(prog.intermediate().clone())
    A.check(L.lib().vlp_debug_route(0, 0))
    a, b = rows
    diff = (a != b).any(dim=1)
    used = (a != 0).any(dim=1) | (b != 0).any(dim=1)
    print(f"config {cfg}: {int(used.sum())} intermediate gate-output rows written, {int(diff.sum())} differ between the "
          f"engines; result rows equal: {bool(torch.equal(outs[0], outs[1]))}", flush=True)
    del rows, a, b
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for c in [int(x) for x in (sys.argv[1:] or ["2", "3"])]:
        run(c)
