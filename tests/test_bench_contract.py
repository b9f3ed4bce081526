"""The bench.py JSON contract on CPU: the reference arm (the CPU oracle, `--impl reference`) prints one JSON
line with the keys the driver reads, and exits 0 without work on non-zero ranks (torchrun N > 1); on a GPU, the
N > 1 path of our arm under torchrun with the ranks sharing one GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run({}, "--steps", "1", "--warmup", "0")
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"] == "gate bootstraps/sec and records/sec per query at 1/2/4/8 B200"
    assert d["config"]["workload"] == "cfg3_rect2d_4096"  # the same config as the GPU arm's default line (config 3)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--steps", "1", "--warmup", "0") == []


def test_algorithmic_ops_per_br_is_survey_8d():
    """roofline.frac's numerator follows SURVEY 8(d): 5,040 transforms (25.8 M butterflies) + 7.74 M MACs per BR
    at the stated per-op costs (7 / butterfly, 2 / MAC, 15 / digit coefficient, 19 / lifted coefficient)."""
    sys.path.insert(0, ROOT)
    import bench
    butterflies = 630 * 8 * 5120
    macs = 630 * 12 * 1024
    assert butterflies == 25_804_800 and macs == 7_741_440
    assert bench.alg_ops_per_br() == butterflies * 7 + macs * 2 + 630 * 2048 * (15 + 19) == 239_984_640
    peak, how = bench.int_peak()
    assert how.startswith("measured") and 25_000 < peak < 40_000  # profiles/int_peak_r1.json, Gop/s
    assert 17_000 < bench.fp64_peak() < 19_000  # profiles/fp64_bench_r2.json


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,world", [(2, 2), (5, 2)])
def test_bench_multi_rank_path_on_one_gpu(cfg, world):
    """bench.py's N > 1 path as the driver launches it (torchrun, one process per rank, WORLD_SIZE / RANK /
    LOCAL_RANK from the env) with every rank on cuda:0 over gloo (VLP_BENCH_ONE_GPU_GLOO=1, CPU-staged
    broadcast / gather in dist.sharded_step): records sharded x2, the gathered shard roots combined on rank 0 and
    checked against the plain predicate inside bench.py (config 2), or the NAND batch split over the ranks
    (config 5); rank 0 alone prints one JSON line with n_gpus = world.  The ranks' kernels never wait on one another,
    so sharing one GPU is safe; the timings are not a scaling measurement."""
    env = dict(os.environ, VLP_BENCH_ONE_GPU_GLOO="1")
    args = ["--config", str(cfg), "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    if cfg == 5:
        args += ["--nand", str(1 << 12)]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                        os.path.join(ROOT, "bench.py"), "--gpus", str(world), *args],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["value"] > 0 and d["steps"] == 1
    if cfg == 2:
        assert d["config"]["parallelism"] == f"records sharded x{world}"
        assert d["config"]["br_per_query"] == 132_080
        assert d["e2e"]["value"] > 0
    else:
        assert d["config"]["gates"] == 1 << 12


@pytest.mark.gpu
def test_bench_multi_rank_multi_query_on_one_gpu():
    """SURVEY 8(f) NEXT 2 at G > 1: two ranks (one GPU, gloo, as above) each pack 2 queries against their shard of
    config 2 (vlp_program_create_queries on [first, first + count)), rank 0 gathers the 2 x 2 shard roots and combines
    each query; bench.py checks both queries' decrypted results against the plain predicate."""
    env = dict(os.environ, VLP_BENCH_ONE_GPU_GLOO="1")
    args = ["--config", "2", "--queries", "2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                        os.path.join(ROOT, "bench.py"), "--gpus", "2", *args],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["queries_per_step"] == 2
    assert d["config"]["parallelism"] == "records sharded x2" and d["e2e"]["value"] > 0
