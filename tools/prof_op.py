"""ncu driver: config-2 block once (warm), then ONE op under cudaProfilerStart/Stop.
usage: ncu --profile-from-start off ... python tools/prof_op.py {mlp_fwd|head_fwd|head_bwd|mlp_bwd|step|attn}
(attn: libmst's causal GQA attention forward + backward at Llama3-8B heads, S=8192)"""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_15892_b200 import miniseq as ms
op = sys.argv[1]
if op == 'attn':
    from paper_2407_15892_b200 import attention as A
    Sa, Ha, KVa, hd = 8192, 32, 8, 128
    torch.manual_seed(0)
    q = torch.randn(Sa, Ha * hd, device='cuda').bfloat16()
    k = torch.randn(Sa, KVa * hd, device='cuda').bfloat16()
    v = torch.randn(Sa, KVa * hd, device='cuda').bfloat16()
    do = torch.randn(Sa, Ha * hd, device='cuda').bfloat16()
    o, lse = A.attention_forward(q, k, v, 1, Sa, Ha, KVa)
    A.attention_backward(q, k, v, o, do, lse, 1, Sa, Ha, KVa)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    o, lse = A.attention_forward(q, k, v, 1, Sa, Ha, KVa)
    A.attention_backward(q, k, v, o, do, lse, 1, Sa, Ha, KVa)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sys.exit(0)
S, M = 8192, 8
H, I, V = 4096, 14336, 128256
dev = 'cuda'
torch.manual_seed(0)
X = torch.randn(S, H, device=dev).bfloat16()
Wg, Wu = [(0.02 * torch.randn(H, I, device=dev)).bfloat16() for _ in range(2)]
Wd = (0.02 * torch.randn(I, H, device=dev)).bfloat16()
Wo = (0.02 * torch.randn(H, V, device=dev)).bfloat16()
L = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
mlp, head = ms.MlpWeights(Wg, Wu, Wd), ms.LmHeadWeights(Wo)
plan = ms.make_chunk_plan(S, M)
st, gr = ms.block_step(X, L, mlp, head, M, M)
O, sv = ms.miniseq_mlp_forward(X, mlp, plan)
loss, hs = ms.miniseq_lmhead_forward(O, L, head, plan)
dO, _ = ms.miniseq_lmhead_backward(hs, head, plan, dW_out=gr.W_out)
torch.cuda.synchronize()
prof = torch.cuda.profiler
prof.start()
if op == 'mlp_fwd':
    ms.miniseq_mlp_forward(X, mlp, plan)
elif op == 'head_fwd':
    ms.miniseq_lmhead_forward(O, L, head, plan)
elif op == 'head_bwd':
    ms.miniseq_lmhead_backward(hs, head, plan, dW_out=gr.W_out)
elif op == 'mlp_bwd':
    ms.miniseq_mlp_backward(dO, sv, mlp, plan, grads=ms.MlpGrads(gr.W_gate, gr.W_up, gr.W_down))
else:
    ms.block_step(X, L, mlp, head, M, M, grads=gr, stats=st)
torch.cuda.synchronize()
prof.stop()
