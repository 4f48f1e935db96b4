"""The decoder around the MsT blocks (paper_2407_15892_b200/model.py, SPEC.md
model module :410-469) on the GPU: libmst GEMM / RMSNorm / embedding / MsT
kernels + the library attention kernel, against the fp32 torch reference
(tests/torch_model_ref.py) and the SPEC's model properties.

Tolerances: loss relative 5e-3; every gradient normwise relative 3e-2
(bf16 activations through the residual stream of a 2-layer model; measured
values are printed on failure).  M-consistency and recompute are checked
much tighter (same kernels, same data)."""
import numpy as np
import pytest
import torch

import torch_model_ref as R
from paper_2407_15892_b200 import miniseq as ms
from paper_2407_15892_b200 import model as mdl
from paper_2407_15892_b200 import optim

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / max(float(b.norm()), 1e-30))


def _data(cfg, seed=0, p_ignore=0.1):
    g = torch.Generator().manual_seed(seed)
    tok = torch.randint(0, cfg.V, (cfg.B, cfg.S), generator=g)
    lab = torch.randint(0, cfg.V, (cfg.B, cfg.S), generator=g)
    lab[torch.rand(cfg.B, cfg.S, generator=g) < p_ignore] = -100
    return tok.int().cuda(), lab.int().cuda()


@pytest.mark.parametrize("cfg", [
    mdl.ModelConfig(),                                                   # SPEC desk-scale default (d=64, I=224, V=2048)
    mdl.ModelConfig(d=128, I=448, V=4096, heads=8, G=4, layers=2, S=512, B=2, M_mlp=4, M_head=16),
    mdl.ModelConfig(layers=0, S=128),                                   # embedding + norm + LM-Head
], ids=["desk", "gqa4_b2_mst", "zero_layers"])
def test_model_matches_torch_reference(cfg):
    m = mdl.Model(cfg)
    tok, lab = _data(cfg)
    loss, saved = m.forward(tok, lab)
    grads = m.backward(saved)
    torch.cuda.synchronize()
    rl, rg = R.loss_and_grads(cfg, m.w.named(), tok, lab)
    assert abs(float(loss) - rl) / rl < 5e-3, (float(loss), rl)
    errs = {k: nrel(grads[k], rg[k]) for k in rg}
    assert set(grads) == set(rg)
    assert max(errs.values()) < 3e-2, errs


def test_miniseq_vs_standard_and_recompute():
    """(M_mlp=4, M_head=16) vs (1,1) -> same loss; recompute
    policy on/off -> identical results."""
    base = mdl.ModelConfig(d=128, I=448, V=4096, heads=4, G=2, layers=2, S=512)
    w = mdl.init_weights(base)
    tok, lab = _data(base, 3)
    res = {}
    for name, kw in {"std": dict(M_mlp=1, M_head=1), "mst": dict(M_mlp=4, M_head=16),
                     "mst_rc": dict(M_mlp=4, M_head=16, recompute=True)}.items():
        cfg = mdl.ModelConfig(**{**base.__dict__, **kw})
        m = mdl.Model(cfg, w)
        loss, saved = m.forward(tok, lab)
        res[name] = (float(loss), m.backward(saved))
    assert abs(res["std"][0] - res["mst"][0]) <= 1e-5 * res["std"][0]
    for k in res["std"][1]:
        assert nrel(res["mst"][1][k], res["std"][1][k]) < 2e-3, k
        assert torch.equal(res["mst"][1][k], res["mst_rc"][1][k]), k  # recompute: bitwise
    assert res["mst"][0] == res["mst_rc"][0]


def test_init_weights_spec_properties():
    cfg = mdl.ModelConfig(layers=2)
    a, b = mdl.init_weights(cfg).named(), mdl.init_weights(cfg).named()
    for k in a:
        assert torch.equal(a[k], b[k]), k  # same seed -> bitwise identical
    assert all(torch.all(a[k] == 1.0) for k in a if ".g_" in k or k == "g_final")  # gains exactly 1
    W = mdl.init_weights(mdl.ModelConfig(d=64, I=64)).named()["layers.0.W_gate"].float()
    assert 0.016 <= float(W.std()) <= 0.024  # std 0.02 +- 20% on 4096 elements
    # adding layers does not perturb earlier ones (per-parameter sub-seeds)
    c = mdl.init_weights(mdl.ModelConfig(layers=3)).named()
    assert torch.equal(c["layers.1.W_qkv"], a["layers.1.W_qkv"]) and torch.equal(c["embedding"], a["embedding"])


def test_embedding_grad_sparsity_and_token_range():
    cfg = mdl.ModelConfig(S=128, V=2048)
    m = mdl.Model(cfg)
    tok, lab = _data(cfg, 5)
    loss, saved = m.forward(tok, lab)
    dE = m.backward(saved)["embedding"]
    present = torch.zeros(cfg.V, dtype=torch.bool, device="cuda")
    present[tok.reshape(-1).long()] = True
    rownz = dE.abs().sum(1) > 0
    assert torch.equal(rownz & ~present, torch.zeros_like(rownz))  # nonzero only for present tokens
    assert bool(rownz[present].all())
    bad = tok.clone()
    bad[0, 3] = cfg.V
    with pytest.raises(ms.DataError):
        m.forward(bad, lab)
    # deterministic embedding scatter: bitwise reruns
    assert torch.equal(m.backward(m.forward(tok, lab)[1])["embedding"], dE)


def test_rmsnorm_kernels_against_torch():
    torch.manual_seed(0)
    for n, d in ((1, 8), (37, 64), (1000, 4096), (64, 4104)):
        x = torch.randn(n, d, device="cuda").bfloat16()
        r = torch.randn(n, d, device="cuda").bfloat16()
        g = torch.rand(d, device="cuda") + 0.5
        y, s, rstd = mdl.rmsnorm_forward(x, g, 1e-5, residual=r)
        s_ref = (x.float() + r.float()).bfloat16().float()
        assert torch.equal(s.float(), s_ref)
        sl = s_ref.clone().requires_grad_(True)
        gl = g.clone().requires_grad_(True)
        yr = sl * torch.rsqrt((sl * sl).mean(-1, keepdim=True) + 1e-5) * gl
        assert nrel(y.float(), yr.detach()) < 4e-3
        dy = torch.randn(n, d, device="cuda").bfloat16()
        dres = torch.randn(n, d, device="cuda").bfloat16()
        yr.backward(dy.float())
        dg = torch.zeros(d, device="cuda")
        dx = mdl.rmsnorm_backward(s, g, rstd, dy, dres, dg, False)
        assert nrel(dx.float(), sl.grad + dres.float()) < 4e-3
        assert nrel(dg, gl.grad) < 1e-4
        dg2 = dg.clone()
        mdl.rmsnorm_backward(s, g, rstd, dy, dres, dg2, True)  # accumulate
        assert torch.allclose(dg2, 2 * dg, rtol=1e-4, atol=1e-5)


def test_training_loss_curves_match_across_M():
    """Fig. 4 property: training the same seed/data with
    (M_mlp, M_head) = (1,1) and (4,16) gives (nearly) identical loss curves,
    and the loss goes down."""
    curves = {}
    for M in ((1, 1), (4, 16)):
        cfg = mdl.ModelConfig(d=64, I=224, V=2048, layers=2, S=256, B=2, M_mlp=M[0], M_head=M[1], seed=7)
        m = mdl.Model(cfg)
        opt = optim.AdamW(m.w.named(), optim.OptimConfig(lr=2e-3))
        tok, lab = _data(cfg, 11, p_ignore=0.0)
        losses = []
        for _ in range(10):
            loss, _ = m.train_step(tok, lab, opt)
            losses.append(float(loss))
        curves[M] = losses
    a, b = np.array(curves[(1, 1)]), np.array(curves[(4, 16)])
    assert np.max(np.abs(a - b) / a) < 5e-3, (a, b)
    assert a[-1] < 0.8 * a[0], a
