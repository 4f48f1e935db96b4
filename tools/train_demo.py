"""End-to-end training on the device (dev tool): a Llama-style decoder on
libmst (tcgen05 attention, mini-sequence MLP / LM-Head blocks, device AdamW
with global-norm clipping) learns a synthetic next-token task, standard
(M = 1) and mini-sequence (M_mlp = 4, M_head = 8) blocks side by side from
the same initial weights and batches.  The task: every sequence is an
arithmetic progression mod V with a per-sequence random start and stride
(stride in 1..3), so the next token is predictable from the previous two:
the loss falls from ln V towards 0 only if attention, the MLP and the head
all learn.  Prints one JSON line per logged step.

  python tools/train_demo.py [steps] [log_every]
"""
import json
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_15892_b200 import model as mdl, optim  # noqa: E402


def batch(g, B, S, V):
    start = torch.randint(0, V, (B, 1), generator=g)
    stride = torch.randint(1, 4, (B, 1), generator=g)
    seq = (start + stride * torch.arange(S + 1)) % V
    return seq[:, :-1].int().cuda(), seq[:, 1:].int().cuda()


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 600
    every = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    V, S, B = 512, 256, 4
    runs = {}
    for name, (mm, mh) in {"standard": (1, 1), "mini_sequence": (4, 8)}.items():
        cfg = mdl.ModelConfig(d=256, I=688, V=V, heads=4, G=2, layers=2, S=S, B=B, M_mlp=mm, M_head=mh, seed=3)
        m = mdl.Model(cfg)
        opt = optim.AdamW(m.w.named(), optim.OptimConfig(lr=1e-3, weight_decay=0.0, clip_norm=1.0))
        g = torch.Generator().manual_seed(7)
        hist = []
        t0 = time.time()
        for it in range(1, steps + 1):
            tok, lab = batch(g, B, S, V)
            loss, _ = m.train_step(tok, lab, opt)
            if it == 1 or it % every == 0:
                lv = float(loss)
                hist.append((it, lv))
                print(json.dumps({"run": name, "M_mlp": mm, "M_head": mh, "step": it, "loss": round(lv, 4)}),
                      flush=True)
        torch.cuda.synchronize()
        runs[name] = hist
        print(json.dumps({"run": name, "steps": steps, "seconds": round(time.time() - t0, 1),
                          "first_loss": hist[0][1], "last_loss": hist[-1][1], "ln_V": round(math.log(V), 4)}),
              flush=True)
    a, b = runs["standard"], runs["mini_sequence"]
    print(json.dumps({"max_abs_loss_diff_standard_vs_mini_sequence": max(abs(x[1] - y[1]) for x, y in zip(a, b))}))


if __name__ == "__main__":
    main()
