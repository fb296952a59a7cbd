"""T6 (-m gpu): the multi-GPU shard path through the CUDA kernels with world_size
2 on ONE GPU -- each rank (a separate process, gloo for the rendezvous) builds bench.py's job for its
fl_shard_range shard of the fixed BASELINE problem and runs it through fl_attn_fwd; every rank's output
block must equal the same block of the single-process run bit for bit (P10: per-(b,h) work is the same
code on the same data, whatever the rank count)."""
import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, variant, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    job = bench.make_job(variant, rank, world, dev, with_host=False)
    for c in job.calls:
        c.fn()
    torch.cuda.synchronize()
    torch.save([(blk, out.cpu()) for blk, out in job.outputs], os.path.join(outdir, f"{variant}_{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["causal", "document", "diff", "evo_col", "evo_row"])
def test_two_ranks_on_one_gpu_equal_single_process(tmp_path, variant):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    world = 2
    ctx = mp.get_context("spawn")
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, variant, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    dev = torch.device("cuda", 0)
    job = bench.make_job(variant, 0, 1, dev, with_host=False)
    for c in job.calls:
        c.fn()
    torch.cuda.synchronize()
    (_, full), = [(b, o.cpu()) for b, o in job.outputs]
    covered = 0
    for r in range(world):
        for blk, out in torch.load(os.path.join(tmp_path, f"{variant}_{r}.pt")):
            if variant.startswith("evo"):
                u0, u1 = blk
                ref = full[:, u0:u1]                   # [B, G, H, S, c] views: G = MSA rows / residue columns
            else:
                g0, g1, b0, b1 = blk
                grp = full.shape[1] // (bench.VARIANTS[variant].get("Hkv") or full.shape[1])
                ref = full[b0:b1, g0 * grp:g1 * grp]
            assert torch.equal(out, ref), f"{variant}: rank {r} block {blk} differs from the single-process output"
            covered += out.numel()
    assert covered == full.numel()
