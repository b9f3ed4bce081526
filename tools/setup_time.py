"""Developer tool: encrypted-DB setup time for a config, host (vlp_pubkeygen + vlp_server_encrypt_db, then
H2D) vs device (vlp_encrypt_db_device)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_12761_b200 import api as A
from synth import make_workload

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = make_workload(cfg)
keys = A.Keys(wl.key_seed)
m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
torch.zeros(1, device="cuda:0")
t0 = time.time()
db_h = A.to_device(keys.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1))
torch.cuda.synchronize()
t1 = time.time()
db_d = A.encrypt_db_device(keys, m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1)
torch.cuda.synchronize()
t2 = time.time()
same = bool(torch.equal(db_h, db_d))
print(f"config {cfg}: {db_h.shape[0]} DB ciphertexts; host {t1 - t0:.2f} s, device {t2 - t1:.2f} s, "
      f"byte-identical {same}, host cores {os.cpu_count()}")
