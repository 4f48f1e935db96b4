"""Run `steps` config-2 block steps with MST_TUNE knobs (dev tool: ncu target).
usage: MST_TUNE=k=v,... python tools/one_step.py [steps]"""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
S, M, H, I, V = 8192, 8, 4096, 14336, 128256
torch.manual_seed(0)
X = torch.randn(S, H, device='cuda').bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device='cuda')).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device='cuda')).bfloat16()
Wo = (0.02 * torch.randn(H, V, device='cuda')).bfloat16()
L = torch.randint(0, V, (S,), device='cuda', dtype=torch.int32)
ctx = ms.Context.get(0)
for kv in filter(None, os.environ.get('MST_TUNE', '').split(',')):
    k, v = kv.split('=')
    ctx.set_tuning(k, int(v))
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
st, gr = ms.block_step(X, L, mlp, head, M, M)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
print("loss", float(st[2]))
