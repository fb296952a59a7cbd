"""Multi-GPU host logic on CPU (world_size 2, gloo): the path shards into independent batch x head
units with no exchange step, so what must hold is
  * every rank regenerates exactly its slice of the global seeded inputs (P10),
  * fl_shard_range partitions the units,
  * the per-rank results, gathered, equal the single-process result bit for bit,
  * the bench's max-over-ranks timing reduction and one-line-per-job output under torchrun.
The per-rank compute here is the oracle (no GPU on this box); on the GPU box each rank runs the
same shard through fl_attn_fwd (bench.py)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    cfg = dict(B=2, H=2, S=96, D=16, mask="causal")
    host = bench.dense_inputs(cfg, rank, world)                  # this rank's batch slice
    out, lse = oracle.attn(host["q"], host["k"], host["v"], mask="causal")
    t = torch.from_numpy(out).reshape(cfg["B"], cfg["H"], cfg["S"], cfg["D"])
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)                                    # off the clock: validation only
    mx = bench.max_over_ranks([float(rank + 1), 10.0 - rank], "cpu", world)
    if rank == 0:
        q_out.put((torch.cat(parts, 0).numpy(), mx))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_process():
    import bench
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, mx = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = dict(B=2, H=2, S=96, D=16, mask="causal")
    full = bench.dense_inputs(dict(cfg, B=cfg["B"] * world), 0, 1)
    ref, _ = oracle.attn(full["q"], full["k"], full["v"], mask="causal")
    assert np.array_equal(gathered.reshape(ref.shape), ref)
    assert mx == [2.0, 10.0]                                      # max over ranks, element-wise


def test_rank_slices_match_global_tensors():
    import bench
    from paper_2511_02043_b200 import synth
    cfg = dict(B=2, H=3, S=40, D=8, diff=True)
    g = bench.dense_inputs(dict(cfg, B=4), 0, 1)
    for r in range(2):
        s = bench.dense_inputs(cfg, r, 2)
        for n in ("q", "k", "v"):
            assert torch.equal(s[n], g[n][r * 2:(r + 1) * 2]), n
    offs = synth.doc_offsets(4, 512, 12, seed=1)
    c2 = dict(B=2, S=512, n_docs=12)
    assert np.array_equal(bench.doc_offsets_for(c2, 1, 2), offs[2:4])
    qg, kg = synth.clustered_qk((4, 2, 300, 16), (4, 2, 300, 16), seed=2)
    q1, k1 = synth.clustered_qk((4, 2, 300, 16), (4, 2, 300, 16), seed=2, b_range=(2, 4))
    assert torch.equal(q1, qg[2:]) and torch.equal(k1, kg[2:])
    ev = dict(evo="row", B=1, Ns=8, Nr=16, H=2, D=32)
    e_all = bench.evo_inputs(dict(ev, B=2), 0, 1)
    e1 = bench.evo_inputs(ev, 1, 2)
    for n in ("Q", "K", "V", "G", "pb"):
        assert torch.equal(e1[n], e_all[n][1:2]), n


def test_shard_range_covers_units_contiguously():
    from paper_2511_02043_b200 import _lib
    pytest.importorskip("ctypes")
    if not os.path.exists(_lib.SO_PATH):
        pytest.skip("library not built")
    from paper_2511_02043_b200 import fl
    for units in (1, 7, 128, 1000):
        for world in (1, 2, 3, 8):
            spans = [fl.shard_range(units, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == units
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def test_reference_arm_under_torchrun_prints_one_line():
    """bench.py --impl reference launched exactly as the driver does for N=2 (gloo, no GPU here):
    rank 0 prints one JSON line, rank 1 exits 0 without work."""
    env = dict(os.environ, FL_REF_BUDGET_S="0.5", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--variant", "evo_col"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
