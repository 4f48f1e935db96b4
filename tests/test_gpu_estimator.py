"""estimator.predict_peak(convention="repo") against tracked device
allocations of model.py ("Tracker agreement:
within 10%"): one train step (forward, backward, deferred AdamW) of a
Llama-style decoder at widths where the MLP / LM-Head intermediates dominate,
with standard and mini-sequence blocks, with and without per-layer
recompute; the measured peak is torch's allocator high-water mark above the
pre-model baseline (libmst's context workspace released first)."""
import pytest
import torch

from paper_2407_15892_b200 import estimator as E
from paper_2407_15892_b200 import miniseq as ms
from paper_2407_15892_b200 import model as mdl
from paper_2407_15892_b200 import optim

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mm,mh,recompute", [(1, 1, False), (4, 16, False), (1, 1, True), (4, 16, True)])
def test_predict_peak_matches_tracked_model_allocations(mm, mh, recompute):
    d, I, V, heads, G, L, S = 1024, 3584, 32000, 8, 2, 4, 8192
    ctx = ms.Context.get(0)
    ctx._ws = None
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    cfg = mdl.ModelConfig(d=d, I=I, V=V, heads=heads, G=G, layers=L, S=S, B=1, M_mlp=mm, M_head=mh,
                          recompute=recompute)
    m = mdl.Model(cfg)
    opt = optim.AdamW(m.w.named(), optim.OptimConfig(lr=1e-4))
    g = torch.Generator(device="cuda").manual_seed(0)
    tok = torch.randint(0, V, (1, S), device="cuda", generator=g)
    lab = torch.randint(0, V, (1, S), device="cuda", generator=g)
    m.train_step(tok, lab, opt)
    torch.cuda.synchronize()
    measured = torch.cuda.max_memory_allocated() - base
    pred = E.predict_peak(d, I, V, heads, G, L, S, 1, mm, mh, recompute, False, convention="repo")
    print(f"M=({mm},{mh}) recompute={recompute}: predicted {pred.total / 2**30:.3f} GiB ({pred.phase}) "
          f"measured {measured / 2**30:.3f} GiB, ratio {pred.total / measured:.3f}",
          {k: round(v, 3) for k, v in pred.rows().items()})
    assert abs(pred.total - measured) / measured <= 0.10
    del m, opt
    ctx._ws = None
    torch.cuda.empty_cache()
