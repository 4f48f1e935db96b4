"""HBM roofline of the optimizer kernels at the config-2 block's parameter
count (W_gate, W_up, W_down, W_out: 3HI + HV = 701M parameters) (dev tool).
AdamW moves 30 B/parameter (read w, g, m, v fp32; write w, m, v fp32 and
the bf16 copy); the global-norm pass reads 4 B/parameter.
usage: python tools/optim_bench.py"""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import optim
from bench import load_peaks

H, I, V = 4096, 14336, 128256
dev = 'cuda'
shapes = {"W_gate": (H, I), "W_up": (H, I), "W_down": (I, H), "W_out": (H, V)}
W = {k: (0.02 * torch.randn(*s, device=dev)).bfloat16() for k, s in shapes.items()}
G = {k: 1e-3 * torch.randn(*s, device=dev) for k, s in shapes.items()}
opt = optim.AdamW(W, optim.OptimConfig())
n = sum(w.numel() for w in W.values())
peak = load_peaks()["hbm"]


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_norm = timed(lambda: optim.global_norm_scale(list(G.values()), 1.0, work=opt._work))
t_adam = timed(lambda: optim.adamw_step(G, opt.state, opt.cfg, grad_scale=opt._work.scale))
t_step = timed(lambda: opt.step(G))
res = {
    "params": n,
    "adamw": {"ms": t_adam, "bytes": 30 * n, "gbs": 30 * n / t_adam / 1e6, "frac_of_hbm": 30 * n / t_adam / 1e6 / peak},
    "global_norm": {"ms": t_norm, "bytes": 4 * n, "gbs": 4 * n / t_norm / 1e6, "frac_of_hbm": 4 * n / t_norm / 1e6 / peak},
    "optimizer_step_ms": t_step,
    "hbm_peak_gbs": peak,
}
print(json.dumps(res))
