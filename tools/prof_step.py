"""Minimal driver for ncu: config-2 block_step, W warm-up steps then 1 step."""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
S, M, W = 8192, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 1
H, I, V = 4096, 14336, 128256
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
st, gr = ms.block_step(X, L, mlp, head, M, M)
for _ in range(W):
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
print("loss", float(st[2]))
