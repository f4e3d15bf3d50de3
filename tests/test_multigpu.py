"""Multi-GPU parity of the three sequence-parallel executors over NCCL: the
Python executor (sp.SPAttention), the same with the O return fused into K4's
epilogue (symmetric memory), and the C++ executor (dbsp_sp_attention).  Every
rank computes its home shard; rank 0 compares the gathered result with the
one-GPU kernel.  Skipped on boxes with fewer than two GPUs (this round's pool
has one); run as part of `pytest -m gpu` where more are visible."""
import os
import socket
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, strategy, mode, result_q):
    import torch
    import torch.distributed as dist

    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.attention import sparse_attention
    from paper_2511_23113_b200.sp import NativeSPContext, SPAttention, home_range
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    try:
        dist.barrier()
        H, S, d = 8, 4096, 128
        nb = S // 64
        masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.5, 1.0, 61))
        st = D.parse_strategy(strategy)
        plan = D.plan_dual(masks, st).plan
        g = torch.Generator().manual_seed(62)
        q, k, v = (torch.randn(S, H, d, generator=g).to(torch.bfloat16) for _ in range(3))
        lo, hi = home_range(rank, world, nb)
        qh, kh, vh = (t[lo * 64:hi * 64].contiguous().to(dev) for t in (q, k, v))
        if mode == "native":
            def bcast(b):
                obj = [b]
                dist.broadcast_object_list(obj, src=0)
                return obj[0]
            ctx = NativeSPContext(rank, world, bcast)
            out = ctx(masks, st, plan, qh, kh, vh)
        else:
            sp = SPAttention(masks, st, plan, S, d, rank, world, dev, fuse_return=(mode == "fused"))
            out = sp(qh, kh, vh)
        torch.cuda.synchronize()
        parts = [torch.empty((home_range(r, world, nb)[1] - home_range(r, world, nb)[0]) * 64, H, d,
                             device=dev, dtype=torch.bfloat16) for r in range(world)]
        dist.all_gather(parts, out.contiguous())
        if rank == 0:
            full = torch.cat(parts, 0)
            ref = sparse_attention(q.to(dev), k.to(dev), v.to(dev), masks)
            err = float((full.float() - ref.float()).abs().max())
            result_q.put(err)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["python", "fused", "native"])
def test_sp_executors_over_nccl(mode):
    import torch.multiprocessing as mp
    here = Path(__file__).resolve().parent
    # spawned ranks import this module and the package from the repo
    os.environ["PYTHONPATH"] = os.pathsep.join([str(here.parent), str(here), os.environ.get("PYTHONPATH", "")])
    world = 4 if torch.cuda.device_count() >= 4 else 2
    strategies = ["U2R2", "U4R1", "U1R4"] if world == 4 else ["U2R1", "U1R2"]
    ctx = mp.get_context("spawn")
    for strategy in strategies:
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, strategy, mode, q)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
            assert p.exitcode == 0, f"{mode} {strategy}: rank exited with {p.exitcode}"
        err = q.get(timeout=10)
        # ring merges differ from the one-shot kernel by bf16 rounding only
        assert err <= 2e-2, f"{mode} {strategy}: max-abs {err:.3e} vs one GPU"
