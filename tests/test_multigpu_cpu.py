"""Multi-GPU host logic on CPU (world_size 2-3, gloo): the fixed BASELINE problem partitions into
independent units with no exchange step (§3.1; §3.6) -- h-major (h, b)
units for the LLM configs, MSA rows / residue columns for Evoformer -- so what must hold is
  * fl_shard_range / shard.unit_blocks partition the units exactly once, contiguously,
  * every rank regenerates exactly its slabs of the global seeded inputs (P10),
  * the per-rank results, gathered, equal the single-process result bit for bit,
  * the bench's max-over-ranks / sum-over-ranks reductions and one-line output under torchrun.
Per-rank compute here is the oracle (no GPU on this box); tests/test_multirank_gpu.py runs the same
shards through the CUDA path with two ranks sharing one GPU."""
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
SMALL = dict(B=3, H=4, S=96, D=16, mask="causal")


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
    mine = []
    for blk, host in bench.dense_inputs(SMALL, rank, world):       # this rank's (h, b) rectangles
        out, _ = oracle.attn(host["q"], host["k"], host["v"], mask="causal")
        mine.append((blk, torch.from_numpy(out).reshape(host["q"].shape[0], host["q"].shape[1], SMALL["S"], -1)))
    parts = [None] * world
    dist.all_gather_object(parts, mine)                          # off the clock: validation only
    mx = bench.max_over_ranks([float(rank + 1), 10.0 - rank], "cpu", world)
    sm = bench.sum_over_ranks([float(rank + 1)], "cpu", world)
    if rank == 0:
        q_out.put((parts, mx, sm))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_shards_equal_single_process(world):
    import bench
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, mx, sm = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = bench.dense_inputs(SMALL, 0, 1)[0][1]
    ref, _ = oracle.attn(full["q"], full["k"], full["v"], mask="causal")
    ref = torch.from_numpy(ref).reshape(SMALL["B"], SMALL["H"], SMALL["S"], -1)
    got = torch.full_like(ref, float("nan"))
    for rank_parts in parts:
        for (h0, h1, b0, b1), out in rank_parts:
            assert torch.isnan(got[b0:b1, h0:h1]).all()            # each unit exactly once
            got[b0:b1, h0:h1] = out
    assert torch.equal(got, ref)
    assert mx == [float(world), 10.0] and sm == [world * (world + 1) / 2]


@pytest.mark.parametrize("n_outer,n_inner", [(16, 8), (32, 4), (5, 3), (1, 7), (8, 1)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_unit_blocks_partition_the_grid(n_outer, n_inner, world):
    from paper_2511_02043_b200 import shard
    seen = np.zeros((n_outer, n_inner), dtype=int)
    prev_end = 0
    for r in range(world):
        blocks = shard.unit_blocks(n_outer, n_inner, world, r)
        assert len(blocks) <= 3
        for o0, o1, i0, i1 in blocks:
            assert o0 * n_inner + i0 == prev_end                    # contiguous in the h-major order
            seen[o0:o1, i0:i1] += 1
            prev_end = (o1 - 1) * n_inner + i1
    assert (seen == 1).all() and prev_end == n_outer * n_inner


@pytest.mark.parametrize("world", [2, 4, 8])
def test_baseline_shards_are_single_rectangles(world):
    """At the BASELINE shapes and 1/2/4/8 GPUs every rank's shard is one rectangle: one launch per call."""
    import bench
    for v in ("causal", "diff", "rsa"):
        cfg = bench.VARIANTS[v]
        for r in range(world):
            blocks = bench.dense_blocks(cfg, r, world)
            assert len(blocks) == 1 and blocks[0][1] - blocks[0][0] == cfg["H"] // world


def test_rank_slices_match_global_tensors():
    import bench
    from paper_2511_02043_b200 import synth
    cfg = dict(B=3, H=4, S=40, D=8, diff=True)
    g = bench.dense_inputs(cfg, 0, 1)[0][1]
    for world in (2, 3):
        for r in range(world):
            for (h0, h1, b0, b1), s in bench.dense_inputs(cfg, r, world):
                assert torch.equal(s["q"], torch.cat([g["q"][b0:b1, h0:h1], g["q"][b0:b1, 4 + h0:4 + h1]], 1))
                assert torch.equal(s["k"], torch.cat([g["k"][b0:b1, h0:h1], g["k"][b0:b1, 4 + h0:4 + h1]], 1))
                assert torch.equal(s["v"], g["v"][b0:b1, h0:h1])
    gq = dict(B=2, H=8, Hkv=2, S=24, D=8)
    g = bench.dense_inputs(gq, 0, 1)[0][1]
    for r in range(2):
        for (g0, g1, b0, b1), s in bench.dense_inputs(gq, r, 2):   # GQA: whole KV groups per rank
            assert torch.equal(s["q"], g["q"][b0:b1, g0 * 4:g1 * 4]) and torch.equal(s["k"], g["k"][b0:b1, g0:g1])
    doc = dict(B=4, H=2, S=512, n_docs=12, mask="document")
    offs = synth.doc_offsets(4, 512, 12, seed=1)
    assert np.array_equal(bench.block_variant_kw(doc, (0, 2, 1, 3))[1], offs[1:3])
    al = dict(B=1, H=16, S=8, D=8, mod="alibi")
    kw, _ = bench.block_variant_kw(al, (4, 8, 0, 1))
    assert np.array_equal(kw["alibi_slopes"], synth.alibi_slopes(16)[4:8])   # global heads' slopes (G2)
    for kind in ("row", "col"):
        ev = dict(evo=kind, B=1, Ns=8, Nr=6, H=2, D=32)
        e_all = bench.evo_inputs(ev, 0, 1)
        for r in range(3):
            u0, u1 = bench.evo_range(ev, r, 3)
            e1 = bench.evo_inputs(ev, r, 3)
            for n in ("Q", "K", "V", "G"):
                want = e_all[n][:, u0:u1] if kind == "row" else e_all[n][:, :, u0:u1]
                assert torch.equal(e1[n], want), (kind, n)
            if kind == "row":
                assert torch.equal(e1["pb"], e_all["pb"])            # pair bias replicated
    rq = dict(rsa="prefill", B=2, H=4, S=300, D=16, topk=2)
    qg, kg, vg = bench.rsa_block_inputs(rq, (0, 4, 0, 2))
    q1, k1, v1 = bench.rsa_block_inputs(rq, (1, 3, 1, 2))
    assert torch.equal(q1, qg[1:2, 1:3]) and torch.equal(k1, kg[1:2, 1:3]) and torch.equal(v1, vg[1:2, 1:3])


def test_shard_range_covers_units_contiguously():
    from paper_2511_02043_b200 import _lib
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
    rank 0 prints one JSON line, rank 1 exits 0 without work; ms_per_step is the measured sample time."""
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
    assert 0 < d["ms_per_step"] < 60_000 and d["full_step_ms_extrapolated"] >= d["ms_per_step"]
