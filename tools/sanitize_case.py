"""Developer tool: a small run of every kernel path for compute-sanitizer (one tool per invocation):
a NAND level of 745 gates (one whole 5-bootstrap wave + a latency-mode tail), a MUX batch of 7 (tail
only), a debug key switch of 17 rows, and config 1 end to end; checks the decrypted results."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_12761_b200 import _lib as L
from paper_2506_12761_b200 import api as A
from synth import make_workload, nand_inputs
from synth.workloads import expected_result

keys = A.Keys(77)
srv = A.Server(keys, 0)
a_bits, b_bits = nand_inputs(745, 3)
a = A.to_device(keys.encrypt_bits(a_bits, 5, 0))
b = A.to_device(keys.encrypt_bits(b_bits, 5, 745))
out = torch.zeros((745, 632), dtype=torch.int32, device="cuda:0")
srv.gate_batch(L.NAND, a, b, out)
torch.cuda.synchronize()
assert np.array_equal(keys.decrypt_bits(A.to_host(out)), 1 - (a_bits & b_bits))
c_bits = nand_inputs(7, 4)[0]
o7 = torch.zeros((7, 632), dtype=torch.int32, device="cuda:0")
srv.gate_batch(L.MUX, a[:7], b[:7], o7, c_dev=A.to_device(keys.encrypt_bits(c_bits, 6, 0)))
torch.cuda.synchronize()
assert np.array_equal(keys.decrypt_bits(A.to_host(o7)), np.where(a_bits[:7] == 1, b_bits[:7], c_bits))
rng = np.random.default_rng(1)
nl = rng.integers(0, 2 ** 32, (17, 1028), dtype=np.uint64).astype(np.uint32)
srv.debug_keyswitch(A.to_device(nl))
torch.cuda.synchronize()
wl = make_workload(1)
m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
q = A.to_device(keys.encrypt_query(m, wl.query, 7))
db = A.to_device(keys.encrypt_db(m, wl.records, wl.payloads, pk_seed=9))
r = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
srv.eval(m, q, db, r)
torch.cuda.synchronize()
assert keys.decrypt_value(A.to_host(r)) == expected_result(wl)
print("sanitize case ok")
