"""bench.py's N>1 code path on one GPU: two ranks (gloo, both on cuda:0 --
the MST_SAME_DEVICE mode of bench.py) run parallel.sp_block_step_fused on
their sequence shards with the gradient-slab all-reduces, and must equal the
single-process block step over the whole sequence:
dX bitwise (same 256-row chunks, same global dlogits scale), loss and dW
within fp32 reassociation; every gradient row is reduced exactly once."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, H, I, V, M_RANK = 2048, 256, 512, 4096, 4


def _inputs():
    g = torch.Generator().manual_seed(99)
    X = torch.randn(N, H, generator=g).bfloat16()
    W = [(0.05 * torch.randn(*s, generator=g)).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (N,), generator=g, dtype=torch.int32)
    L[:300] = -100  # rank 0 holds far fewer valid labels than rank 1
    L[::13] = -100
    return X, W, L


def _worker(rank, world, port, slabs, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_15892_b200 import miniseq as ms
        from paper_2407_15892_b200.parallel import GpuOps, shard_rows, sp_block_step_fused

        X, W, L = _inputs()
        s, e = shard_rows(N, world, rank)
        dev = torch.device("cuda", 0)
        Xs, Ls = X[s:e].to(dev), L[s:e].to(dev)
        Wd = [w.to(dev) for w in W]
        grads = ms.alloc_block_grads(e - s, H, I, V, dev)
        r = sp_block_step_fused(GpuOps(), Xs, Ls, tuple(Wd[:3]), Wd[3], M_RANK, M_RANK, grads, slabs=slabs)
        torch.cuda.synchronize()
        ret[rank] = dict(loss=float(r.loss), dX=r.dX.cpu(), dWg=r.dW_gate.cpu(), dWu=r.dW_up.cpu(),
                         dWd=r.dW_down.cpu(), dWo=r.dW_out.cpu())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("slabs", [1, 4])
def test_two_rank_sequence_parallel_equals_single_gpu(slabs):
    from paper_2407_15892_b200 import miniseq as ms

    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), slabs, ret), nprocs=world, join=True)
    X, W, L = _inputs()
    dev = torch.device("cuda", 0)
    Wd = [w.to(dev) for w in W]
    st, gr = ms.block_step(X.to(dev), L.to(dev), ms.MlpWeights(*Wd[:3]), ms.LmHeadWeights(Wd[3]), world * M_RANK,
                           world * M_RANK)
    torch.cuda.synchronize()
    ref_loss = float(st[2])
    dX = torch.cat([ret[r]["dX"] for r in range(world)])
    assert torch.equal(dX, gr.dX.cpu())  # same chunks, same global scale: bitwise rows
    for r in range(world):
        assert abs(ret[r]["loss"] - ref_loss) <= 1e-6 * abs(ref_loss)
        for k, t in (("dWg", gr.W_gate), ("dWu", gr.W_up), ("dWd", gr.W_down), ("dWo", gr.W_out)):
            ref = t.cpu().double()
            err = float((ret[r][k].double() - ref).norm() / ref.norm())
            assert err <= 1e-5, (r, k, err)
        assert torch.equal(ret[r]["dWo"], ret[0]["dWo"])  # every rank holds the same reduced gradient


def test_bench_multi_rank_path_runs():
    """bench.py itself under torchrun with two ranks on one GPU (MST_SAME_DEVICE=1,
    gloo): the N>1 code path (global valid count, slab all-reduces, max-over-ranks
    timing, e2e with dX copied back) runs and prints one JSON line from rank 0."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(__import__("os").environ, MST_SAME_DEVICE="1", MST_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--seq", "2048", "--no-max-seq"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_tokens"] == 4096 and d["value"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == 4 + 2048 * 4096 * 2
    assert "slab" in d["config"]["schedule"]
