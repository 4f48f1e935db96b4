"""Determinism stress (dev tool): the block step is bitwise reproducible, so
any rare race in the engine's hand-offs (tile ring, TMEM, stage barriers)
shows up as a step whose outputs differ from the first.  Runs config 2 for
`steps` steps and a rotation of small ragged shapes, comparing every step's
loss, dX and dW bytes against the first run of the same shape.
usage: python tools/stress_determinism.py [steps]"""
import json, sys, time, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms


def outputs(st, gr):
    return [t.clone() for t in (st[:3], gr.dX, gr.W_gate, gr.W_up, gr.W_down, gr.W_out)]


def same(a, b):  # bitwise, on the device
    return all(torch.equal(x.view(torch.uint8), y.view(torch.uint8)) for x, y in zip(a, b))


def make(S, H, I, V, seed):
    g = torch.Generator(device='cuda').manual_seed(seed)
    X = torch.randn(S, H, device='cuda', generator=g, dtype=torch.bfloat16)
    W = [(0.02 * torch.randn(*s, device='cuda', generator=g)).bfloat16() for s in ((H, I), (H, I), (I, H), (H, V))]
    L = torch.randint(0, V, (S,), device='cuda', generator=g, dtype=torch.int32)
    L[::13] = -100
    return X, L, ms.MlpWeights(*W[:3]), ms.LmHeadWeights(W[3])


steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
shapes = [(8192, 4096, 14336, 128256, 8), (777, 512, 1376, 5000, 3), (300, 256, 688, 4096, 4), (1024, 128, 256, 520, 16)]
data = {s: make(*s[:4], seed=i) for i, s in enumerate(shapes)}
ref, grads, stats, bad, n = {}, {}, {}, 0, 0
t0 = time.time()
for it in range(steps):
    s = shapes[0] if it % 2 == 0 else shapes[1 + (it // 2) % (len(shapes) - 1)]
    X, L, mlp, head = data[s]
    st, gr = ms.block_step(X, L, mlp, head, s[4], s[4], grads=grads.get(s), stats=stats.get(s))
    grads[s], stats[s] = gr, st
    n += 1
    if s not in ref:
        ref[s] = outputs(st, gr)
    elif not same(outputs(st, gr), ref[s]):
        bad += 1
        print(json.dumps({"step": it, "shape": s, "mismatch": True}), flush=True)
print(json.dumps({"steps": n, "mismatches": bad, "shapes": len(shapes), "seconds": time.time() - t0}), flush=True)
