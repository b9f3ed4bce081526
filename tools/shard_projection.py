"""Developer tool (one GPU): the per-GPU work of the G-GPU record sharding measured on one B200 --
every shard of config 3 evaluated down to its root (the same vlp_server_eval a rank runs), then rank 0's
vlp_server_combine of the G roots; the slowest shard + the combine is the device time a G-GPU query would take
without the collectives (an 81 KB broadcast and a G x 32 x 2.5 KB gather, microseconds over NVLink).  Checks that the
combined result decrypts to the predicate.  No multi-GPU box was available; this is a projection, not a scaling run.
    python tools/shard_projection.py [config] [G ...]   (default: 3  2 4 8)"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import api as A  # noqa: E402
from paper_2506_12761_b200.dist import shard_range  # noqa: E402
from synth import make_workload  # noqa: E402
from synth.workloads import expected_result  # noqa: E402

CONFIG_BR = {2: 132080, 3: 1060832, 4: 6750176}


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    args = [int(x) for x in sys.argv[1:]]
    cfg = args[0] if args else 3
    gs = args[1:] or [2, 4, 8]
    wl = make_workload(cfg)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    q = A.to_device(keys.encrypt_query(m, wl.query, 7))
    pk = A.pubkeygen_device(keys, m, wl.key_seed + 1, 0, wl.M)
    db = A.server_encrypt_db_device(m, pk, wl.records, wl.payloads)
    per = A.record_cts(m)
    full = A.Program.velopir(srv, m)
    out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    full.eval(q, db, out)
    t1 = timed(lambda: full.eval(q, db, out))
    br = CONFIG_BR.get(cfg, full.info.br)
    print(f"config {cfg} ({wl.name}) on 1 GPU: {t1:.0f} ms per query, {br / t1 * 1e3:.0f} BR/s", flush=True)
    for G in gs:
        roots = torch.zeros((G * wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        shard_ms = []
        for r in range(G):
            first, count = shard_range(wl.M, G, r)
            prog = A.Program.velopir(srv, m, first, count)
            part = roots[r * wl.l_S:(r + 1) * wl.l_S]
            dbs = db[first * per:(first + count) * per]
            prog.eval(q, dbs, part)
            shard_ms.append(timed(lambda: prog.eval(q, dbs, part)))
            del prog
        comb = A.Program.combine(srv, m, G)
        comb.eval(roots, None, out)
        tc = timed(lambda: comb.eval(roots, None, out))
        ok = keys.decrypt_value(A.to_host(out)) == expected_result(wl)
        tg = max(shard_ms) + tc
        print(f"G = {G}: shard {min(shard_ms):.0f}-{max(shard_ms):.0f} ms, combine {tc:.1f} ms -> {tg:.0f} ms per query, "
              f"projected {br / tg * 1e3:.0f} BR/s ({t1 / tg:.2f}x, {t1 / tg / G * 100:.0f} % of linear), "
              f"predicate {'OK' if ok else 'WRONG'}", flush=True)


if __name__ == "__main__":
    main()
