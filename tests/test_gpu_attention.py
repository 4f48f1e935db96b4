"""The tcgen05 causal GQA attention (csrc/attention.cu, attention.py) against
an fp32 reference of the same math (torch SDPA in fp32 on the same bf16
inputs), forward (o, lse) and backward (dq, dk, dv).

Tolerances (normwise relative): o 1e-2 (bf16 output, bf16 P in the PV GEMM),
lse 1e-4 absolute per row relative to |lse|, dq / dk / dv 2e-2 (bf16 P and dS
operands); reruns bitwise (no atomics)."""
import pytest
import torch
import torch.nn.functional as F

from paper_2407_15892_b200 import attention as A

pytestmark = pytest.mark.gpu

SHAPES = [  # (B, S, heads, kv_heads, hd)
    (1, 128, 4, 4, 64),
    (2, 200, 8, 2, 128),
    (1, 1000, 4, 1, 16),
    (1, 1, 2, 2, 64),
    (3, 129, 4, 2, 32),
    (1, 513, 8, 4, 96),
    (1, 4096, 32, 8, 128),
]


def rel(a, b):
    """Normwise relative error, with a floor of 1e-3 per element RMS for
    gradients that vanish exactly (S = 1: dq = 0 in exact arithmetic)."""
    a, b = a.detach().float(), b.detach().float()
    return float((a - b).norm() / b.norm().clamp_min(1e-3 * b.numel() ** 0.5))


def _ref(q, k, v, B, S, H, KV, hd, do=None):
    """fp32 reference: [B*S, H*hd] token-major -> SDPA [B, H, S, hd]."""
    qf = q.float().reshape(B, S, H, hd).transpose(1, 2).detach().requires_grad_(True)
    kf = k.float().reshape(B, S, KV, hd).transpose(1, 2).detach().requires_grad_(True)
    vf = v.float().reshape(B, S, KV, hd).transpose(1, 2).detach().requires_grad_(True)
    rep = H // KV
    kr, vr = kf.repeat_interleave(rep, dim=1), vf.repeat_interleave(rep, dim=1)
    scores = (qf @ kr.transpose(-1, -2)) / hd ** 0.5
    mask = torch.ones(S, S, dtype=torch.bool, device=q.device).triu(1)
    scores = scores.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(scores, dim=-1)
    o = torch.softmax(scores, dim=-1) @ vr
    out = {"o": o.transpose(1, 2).reshape(B * S, H * hd), "lse": lse}
    if do is not None:
        o.backward(do.float().reshape(B, S, H, hd).transpose(1, 2))
        out.update(dq=qf.grad.transpose(1, 2).reshape(B * S, H * hd),
                   dk=kf.grad.transpose(1, 2).reshape(B * S, KV * hd),
                   dv=vf.grad.transpose(1, 2).reshape(B * S, KV * hd))
    return out


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "B{}_S{}_H{}_KV{}_hd{}".format(*s))
def test_attention_matches_fp32_reference(shape):
    B, S, H, KV, hd = shape
    torch.manual_seed(S + H)
    N = B * S
    q = torch.randn(N, H * hd, device="cuda").bfloat16()
    k = torch.randn(N, KV * hd, device="cuda").bfloat16()
    v = torch.randn(N, KV * hd, device="cuda").bfloat16()
    do = torch.randn(N, H * hd, device="cuda").bfloat16()
    o, lse = A.attention_forward(q, k, v, B, S, H, KV)
    dq, dk, dv = A.attention_backward(q, k, v, o, do, lse, B, S, H, KV)
    torch.cuda.synchronize()
    ref = _ref(q, k, v, B, S, H, KV, hd, do)
    errs = dict(o=rel(o, ref["o"]), lse=float(((lse - ref["lse"]).abs() / ref["lse"].abs().clamp_min(1)).max()),
                dq=rel(dq, ref["dq"]), dk=rel(dk, ref["dk"]), dv=rel(dv, ref["dv"]))
    print(shape, {k_: "%.2e" % v_ for k_, v_ in errs.items()})
    assert errs["o"] <= 1e-2 and errs["lse"] <= 1e-4
    for k_ in ("dq", "dk", "dv"):
        assert errs[k_] <= 2e-2, k_
    o2, lse2 = A.attention_forward(q, k, v, B, S, H, KV)
    g2 = A.attention_backward(q, k, v, o2, do, lse2, B, S, H, KV)
    assert torch.equal(o, o2) and torch.equal(lse, lse2)
    for x, y in zip((dq, dk, dv), g2):
        assert torch.equal(x, y)  # deterministic: no atomics


def test_attention_reads_fused_qkv_slices_in_place():
    """The decoder's fused [N, d + 2 d/G] qkv buffer: q, k, v are column
    slices (row stride d + 2 d/G); dq, dk, dv land in slices of one buffer."""
    B, S, H, KV, hd = 2, 300, 8, 2, 64
    d, kv = H * hd, KV * hd
    torch.manual_seed(0)
    qkv = torch.randn(B * S, d + 2 * kv, device="cuda").bfloat16()
    q, k, v = qkv[:, :d], qkv[:, d:d + kv], qkv[:, d + kv:]
    o, lse = A.attention_forward(q, k, v, B, S, H, KV)
    oc, lsec = A.attention_forward(q.contiguous(), k.contiguous(), v.contiguous(), B, S, H, KV)
    assert torch.equal(o, oc) and torch.equal(lse, lsec)
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    A.attention_backward(q, k, v, o, do, lse, B, S, H, KV, dq=dqkv[:, :d], dk=dqkv[:, d:d + kv], dv=dqkv[:, d + kv:])
    ref = A.attention_backward(q.contiguous(), k.contiguous(), v.contiguous(), o, do, lse, B, S, H, KV)
    assert torch.equal(dqkv[:, :d], ref[0]) and torch.equal(dqkv[:, d:d + kv], ref[1])
    assert torch.equal(dqkv[:, d + kv:], ref[2])


def test_attention_autograd_function():
    B, S, H, KV, hd = 1, 256, 4, 2, 64
    torch.manual_seed(2)
    q = torch.randn(B * S, H * hd, device="cuda").bfloat16().requires_grad_(True)
    k = torch.randn(B * S, KV * hd, device="cuda").bfloat16().requires_grad_(True)
    v = torch.randn(B * S, KV * hd, device="cuda").bfloat16().requires_grad_(True)
    o = A.CausalAttention.apply(q, k, v, B, S, H, KV)
    do = torch.randn_like(o)
    o.backward(do)
    ref = _ref(q.detach(), k.detach(), v.detach(), B, S, H, KV, hd, do)
    assert rel(o, ref["o"]) <= 1e-2
    assert rel(q.grad, ref["dq"]) <= 2e-2 and rel(k.grad, ref["dk"]) <= 2e-2 and rel(v.grad, ref["dv"]) <= 2e-2


def test_attention_rejects_bad_arguments():
    from paper_2407_15892_b200 import miniseq as ms

    q = torch.randn(128, 4 * 12, device="cuda").bfloat16()  # hd = 12: not a multiple of 8
    with pytest.raises(ms.ShapeError):
        A.attention_forward(q, q[:, :12 * 2].contiguous(), q[:, :24].contiguous(), 1, 128, 4, 2)
    q = torch.randn(128, 64, device="cuda").bfloat16()
    with pytest.raises(ms.ConfigError):  # heads not a multiple of kv_heads
        A.attention_forward(q, q[:, :48].contiguous(), q[:, :48].contiguous(), 1, 128, 4, 3)


@pytest.mark.parametrize("hd", [128, 64, 96])
def test_backward_issue_orders_bitwise_equal(hd):
    """Every backward issue order (tuning attn_bwd_order: dK/dV next scores
    under the dS pass, dQ's dS over S) and the MMA completion-wait knob only
    move when GEMMs are issued, not what they accumulate: dq / dk / dv are
    bitwise equal to order 0 over several kv / q tiles (ring wrap-around,
    GQA 4)."""
    from paper_2407_15892_b200 import miniseq as ms

    ctx = ms.Context.get(0)
    torch.manual_seed(11)
    S, H, KV = 900, 8, 2
    q = torch.randn(S, H * hd, device="cuda").bfloat16()
    k = torch.randn(S, KV * hd, device="cuda").bfloat16()
    v = torch.randn(S, KV * hd, device="cuda").bfloat16()
    do = torch.randn(S, H * hd, device="cuda").bfloat16()
    o, lse = A.attention_forward(q, k, v, 1, S, H, KV)
    try:
        ctx.set_tuning("attn_bwd_order", 0)
        ref = [t.clone() for t in A.attention_backward(q, k, v, o, do, lse, 1, S, H, KV)]
        for order in (1, 2, 3):
            for inorder in (0, 1):
                ctx.set_tuning("attn_bwd_order", order)
                ctx.set_tuning("attn_inorder", inorder)
                got = A.attention_backward(q, k, v, o, do, lse, 1, S, H, KV)
                for name, a, b in zip(("dq", "dk", "dv"), got, ref):
                    assert torch.equal(a, b), (order, inorder, name)
    finally:
        ctx.set_tuning("attn_bwd_order", 3)
        ctx.set_tuning("attn_inorder", 0)
