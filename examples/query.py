"""End-to-end VeLoPIR query on one B200 through the C ABI (client and server on one machine).

    python examples/query.py [--records 256] [--mode intv|cov|idm]

Client: keygen, PubKeyGen, query encryption, decryption -- all from OS randomness (the *_secure calls;
the seeded calls are the reproducible test / benchmark mode).  Server: evaluation key upload, ServerEnc (from the
client's public-key samples only), server_eval.  The result is checked against the plaintext predicate.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_12761_b200 import _lib as L
from paper_2506_12761_b200 import api as A


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=256)
    ap.add_argument("--mode", default="intv", choices=["intv", "cov", "idm"])
    args = ap.parse_args()
    rng = np.random.default_rng(1)
    M, l_I, l_S = args.records, 16, 16
    if args.mode == "intv":  # 1-D intervals [lo, hi] (IntV, closed upper bound R12)
        mode, d = L.MODE_INTV, 1
        lo = rng.integers(0, 2 ** 16 - 512, M)
        records = np.stack([lo, lo + rng.integers(16, 512, M)], axis=1).astype(np.uint64)
        query = [int(records[M // 2][0]) + 3]
    elif args.mode == "cov":  # points (paper CoV: coordinate equality)
        mode, d = L.MODE_COV, 2
        records = rng.integers(0, 2 ** 16, (M, 2)).astype(np.uint64)
        query = [int(v) for v in records[7 % M]]
    else:  # identifiers
        mode, d = L.MODE_IDM, 1
        records = rng.choice(2 ** 16, M, replace=False).astype(np.uint64).reshape(M, 1)
        query = [int(records[5 % M][0])]
    payloads = rng.integers(0, 2 ** l_S, M, dtype=np.uint64)
    m = A.meta(mode, M, l_I, l_S, d)

    t0 = time.time()
    keys = A.Keys()                               # client: secret key + evaluation key (OS randomness)
    server = A.Server(keys, device=0)             # server: evk on the GPU (bsk -> FFT / NTT domains)
    db = A.to_device(keys.encrypt_db(m, records, payloads))  # client PubKeyGen (OS randomness) + server ServerEnc
    q = A.to_device(keys.encrypt_query(m, query))            # client: encrypted query (OS randomness)
    out = torch.zeros((l_S, A.CT_STRIDE), dtype=torch.int32, device="cuda:0")
    torch.cuda.synchronize()
    server.eval(m, q, db, out)                    # first call compiles and caches the level schedule
    torch.cuda.synchronize()
    t1 = time.time()
    server.eval(m, q, db, out)                    # server_eval: every record at once, level by level
    torch.cuda.synchronize()
    t2 = time.time()
    bits, value = keys.decrypt_result(A.to_host(out), l_S)  # client: decrypt_result
    want = 0
    for rec, pay in zip(records.tolist(), payloads.tolist()):
        if mode == L.MODE_INTV:
            hit = rec[0] <= query[0] <= rec[1]
        else:
            hit = list(rec) == query
        want ^= int(pay) if hit else 0
    print(f"{args.mode}: {M} records, setup + first query {t1 - t0:.2f} s, query {1e3 * (t2 - t1):.1f} ms, "
          f"result {value:#x} (expected {want:#x}) {'OK' if value == want else 'MISMATCH'}")
    sys.exit(0 if value == want else 1)


if __name__ == "__main__":
    main()
