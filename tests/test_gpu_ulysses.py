"""Ulysses sequence-parallel decoder on the GPU path:
two ranks (gloo, both on cuda:0 — the box has one GPU; on a multi-GPU node
the same code runs over NCCL) each hold half of one sequence; attention
re-shards with all-to-alls, the MsT blocks run on the shards, the LM-Head
uses the global valid count and the weight gradients are SUM-all-reduced.
Loss and gradients must equal the single-process model within fp32
reassociation (P>1 == P=1)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(d=128, I=448, V=4096, heads=8, G=4, layers=2, B=1, M_mlp=2, M_head=4)
S = 512


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data():
    g = torch.Generator().manual_seed(3)
    tok = torch.randint(0, CFG["V"], (1, S), generator=g).int()
    lab = torch.randint(0, CFG["V"], (1, S), generator=g).int()
    lab[0, :40] = -100  # uneven valid counts across the shards
    return tok, lab


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_15892_b200 import model as mdl

        torch.cuda.set_device(0)
        cfg = mdl.ModelConfig(**CFG, S=S // world)
        w = mdl.init_weights(mdl.ModelConfig(**CFG, S=S))
        m = mdl.Model(cfg, w, group=dist.group.WORLD)
        tok, lab = _data()
        s = S // world
        loss, saved = m.forward(tok[:, rank * s:(rank + 1) * s].cuda(), lab[:, rank * s:(rank + 1) * s].cuda())
        grads = m.backward(saved)
        torch.cuda.synchronize()
        ret[rank] = dict(loss=float(loss), grads={k: v.cpu() for k, v in grads.items()})
    finally:
        dist.destroy_process_group()


def test_ulysses_model_matches_single_process():
    from paper_2407_15892_b200 import model as mdl

    cfg = mdl.ModelConfig(**CFG, S=S)
    m = mdl.Model(cfg)
    tok, lab = _data()
    loss, saved = m.forward(tok.cuda(), lab.cuda())
    ref = {k: v.cpu() for k, v in m.backward(saved).items()}
    ref_loss = float(loss)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), ret), nprocs=2, join=True)
    assert len(ret) == 2
    for r in range(2):
        out = ret[r]
        assert abs(out["loss"] - ref_loss) <= 1e-5 * ref_loss, (out["loss"], ref_loss)
        for k, g in ref.items():
            e = float((out["grads"][k].double() - g.double()).norm() / max(float(g.double().norm()), 1e-30))
            assert e < 2e-3, (r, k, e)
