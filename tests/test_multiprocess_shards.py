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
