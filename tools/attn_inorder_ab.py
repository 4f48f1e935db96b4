"""A/B of the attention forward with and without the MMA completion wait between dependent MMAs (tuning attn_inorder), interleaved rounds (dev tool)."""
import sys, statistics, torch
sys.path.insert(0,'.')
from paper_2407_15892_b200 import attention as A, miniseq as ms
S,H,KV,hd=8192,32,8,128
q=torch.randn(S,H*hd,device='cuda').bfloat16(); k=torch.randn(S,KV*hd,device='cuda').bfloat16(); v=torch.randn(S,KV*hd,device='cuda').bfloat16()
ctx=ms.Context.get(0); fl=2.0*S*S*hd*H
o,lse=A.attention_forward(q,k,v,1,S,H,KV)
res={0:[],1:[]}
for r in range(8):
    for io in ((0,1) if r%2==0 else (1,0)):
        ctx.set_tuning('attn_inorder',io)
        for _ in range(2): A.attention_forward(q,k,v,1,S,H,KV,out=o)
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): A.attention_forward(q,k,v,1,S,H,KV,out=o)
        e1.record(); torch.cuda.synchronize(); res[io].append(e0.elapsed_time(e1)/5)
for io in (0,1): print('inorder',io, fl/statistics.median(res[io])/1e9)
