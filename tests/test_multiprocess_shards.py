"""N > 1 path on CPU (gloo, world size 2): the sharded query protocol of paper_2506_12761_b200.dist
(broadcast query -> per-shard evaluation down to the shard root -> gather -> top tree levels on rank 0)
gives byte-identical ciphertexts to the single-shot evaluation (R15).  The per-shard evaluation here is the
CPU oracle (no GPU in this container); the GPU bench runs the same dist.sharded_step with the library's
programs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from oracle import circuits as C
from oracle import protocol as P
from paper_2506_12761_b200.dist import shard_range, sharded_step

L_I, L_S, M, SEED = 4, 3, 4, 77
RECORDS = [(2, 9), (0, 5), (4, 4), (3, 15)]
PAYLOADS = [5, 3, 6, 1]
QUERY = [4]
FLAGS = C.CONFIG_FLAGS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _encrypt_db(keys, first, count):
    recs, pays = [], []
    for i in range(first, first + count):
        r, p = P.server_enc_record(keys, 555, i, list(RECORDS[i]), PAYLOADS[i], L_I, L_S)
        recs.append(r)
        pays.append(p)
    return recs, pays


def _to_t(cts):
    a = np.zeros((len(cts), 632), np.uint32)
    a[:, :631] = np.stack(cts)
    return torch.from_numpy(a.view(np.int32))


def _from_t(t):
    return [row[:631].copy() for row in t.numpy().view(np.uint32)]


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys = O.OracleKeys(SEED)
    B = C.TfheBackend(keys)
    first, count = shard_range(M, world, rank)
    recs, pays = _encrypt_db(keys, first, count)
    q = _to_t(P.encrypt_query(keys, QUERY, L_I, 7)[0]) if rank == 0 else torch.zeros((L_I, 632), dtype=torch.int32)

    def eval_shard(qt):
        qc = [_from_t(qt)]
        _, _, masked = C.velopir(B, C.MODE_INTV, qc, recs, pays, L_I, 1, L_S, FLAGS, threads=2)
        root = C.hom_sum_tree(B, masked, L_S)
        return _to_t(root)

    def combine(roots):
        rs = _from_t(roots)
        return _to_t(C.hom_sum_tree(B, [rs[g * L_S:(g + 1) * L_S] for g in range(world)], L_S))

    R = sharded_step(q, eval_shard, combine, world, rank)
    if rank == 0:
        np.save(out_path, R.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range():
    assert shard_range(1024, 8, 3) == (384, 128)
    for bad in [(1000, 8), (96, 2), (64, 3)]:
        with pytest.raises(ValueError):
            shard_range(bad[0], bad[1], 0)


def test_two_rank_gloo_shards_equal_single_shot(tmp_path):
    out = str(tmp_path / "R.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    R2 = np.load(out).view(np.uint32)
    keys = O.OracleKeys(SEED)
    recs, pays = _encrypt_db(keys, 0, M)
    q = P.encrypt_query(keys, QUERY, L_I, 7)
    R1, _, _ = C.velopir(C.TfheBackend(keys), C.MODE_INTV, q, recs, pays, L_I, 1, L_S, FLAGS)
    assert np.array_equal(R2[:, :631], np.stack(R1)[:, :631])
    assert P.decrypt_bits(keys, R1) == C.plain_result(C.MODE_INTV, QUERY, RECORDS, PAYLOADS, 1, FLAGS)


# ----------------------------------------------------------------------------------- the library's shard path
def _gpu_worker(rank, world, port, cfg, out_path):
    """One rank of dist.sharded_step with the real library on cuda:0: the rank's shard is built by the device
    preprocessing calls and evaluated by vlp_server_eval; the query broadcast and the root gather are gloo (CPU
    tensors, staged around the device calls); rank 0 runs vlp_server_combine.  The ranks' kernels never wait on one
    another (each evaluates an independent shard), so running them as processes on one GPU is safe."""
    import torch
    from paper_2506_12761_b200 import api as A
    from synth import make_workload
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = make_workload(cfg)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    first, count = shard_range(wl.M, world, rank)
    pk = A.pubkeygen_device(keys, m, wl.key_seed + 1, first, count)
    db = A.server_encrypt_db_device(m, pk, wl.records[first:first + count], wl.payloads[first:first + count])
    nq = wl.l_I * (1 if wl.mode == 2 else wl.d)
    q = torch.from_numpy(keys.encrypt_query(m, wl.query, 7).view(np.int32)) if rank == 0 else \
        torch.zeros((nq, 632), dtype=torch.int32)

    def eval_shard(qc):
        out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        srv.eval(m, qc.to("cuda:0"), db, out, first=first, count=count)
        return out.cpu()

    def combine(roots):
        out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        srv.combine(m, world, roots.to("cuda:0"), out)
        return out.cpu()

    R = sharded_step(q, eval_shard, combine, world, rank)
    if rank == 0:
        np.save(out_path, R.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,world", [(2, 2), (2, 4), (3, 2), (3, 4)])
def test_library_shards_on_ranks_equal_single_shot(tmp_path, cfg, world):
    """SURVEY 8(e) / R15 with the real library: `world` processes each evaluate a contiguous power-of-two shard
    of config `cfg` through dist.sharded_step (broadcast -> vlp_server_eval -> gather to rank 0 ->
    vlp_server_combine); the result is byte-identical to one vlp_server_eval over all records and decrypts to the
    plain predicate."""
    import torch
    from paper_2506_12761_b200 import api as A
    from synth import make_workload
    from synth.workloads import expected_result
    out = str(tmp_path / "R.npy")
    mp.spawn(_gpu_worker, args=(world, _free_port(), cfg, out), nprocs=world, join=True)
    Rg = np.load(out).view(np.uint32)
    wl = make_workload(cfg)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    db = A.encrypt_db_device(keys, m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1)
    q = A.to_device(keys.encrypt_query(m, wl.query, 7))
    R1 = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    srv.eval(m, q, db, R1)
    R1 = A.to_host(R1)
    assert np.array_equal(Rg, R1)
    assert keys.decrypt_value(R1) == expected_result(wl)
