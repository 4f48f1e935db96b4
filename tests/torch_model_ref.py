"""fp32 PyTorch reference of the decoder for the GPU model
tests — TEST INFRASTRUCTURE ONLY.  Same weights (bf16 values upcast), naive
causal grouped-query attention with materialised scores,
RMSNorm eps 1e-5, token-weighted mean cross-entropy over labels != -100,
gradients by autograd.  bf16 rounding is applied where the product stores
bf16 activations (RMSNorm outputs, the residual stream, Q/K/V, attention
output, MLP hidden h and output), so the remaining difference is fp32
accumulation order and the library attention kernel."""
import torch


def _bf(t):
    return t.bfloat16().float()


def _rms(x, g, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g


def forward(cfg, named, tokens, labels):
    """loss (autograd graph over fp32 leaf copies of `named`); returns (loss, leaves)."""
    leaves = {k: v.detach().float().clone().requires_grad_(True) for k, v in named.items()}
    B, S, d, h, G = cfg.B, cfg.S, cfg.d, cfg.heads, cfg.G
    hd, kvh, kv = d // h, h // G, d // G
    x = leaves["embedding"][tokens.reshape(-1).long()]
    for i in range(cfg.layers):
        p = f"layers.{i}."
        a = _bf(_rms(x, leaves[p + "g_attn"], cfg.eps))
        qkv = _bf(a @ leaves[p + "W_qkv"])
        q = qkv[:, :d].reshape(B, S, h, hd).transpose(1, 2)
        k = qkv[:, d:d + kv].reshape(B, S, kvh, hd).transpose(1, 2).repeat_interleave(G, dim=1)
        v = qkv[:, d + kv:].reshape(B, S, kvh, hd).transpose(1, 2).repeat_interleave(G, dim=1)
        sc = (q @ k.transpose(-1, -2)) / hd ** 0.5
        mask = torch.ones(S, S, dtype=torch.bool, device=sc.device).triu(1)
        sc = sc.masked_fill(mask, float("-inf"))
        o = _bf((sc.softmax(-1) @ v).transpose(1, 2).reshape(B * S, d))
        x2 = _bf(x + _bf(o @ leaves[p + "W_o"]))
        b = _bf(_rms(x2, leaves[p + "g_mlp"], cfg.eps))
        hh = _bf(torch.nn.functional.silu(b @ leaves[p + "W_gate"]) * (b @ leaves[p + "W_up"]))
        x = _bf(x2 + _bf(hh @ leaves[p + "W_down"]))
    f = _bf(_rms(x, leaves["g_final"], cfg.eps))
    logits = f @ leaves["W_out"]
    loss = torch.nn.functional.cross_entropy(logits, labels.reshape(-1).long(), ignore_index=-100)
    return loss, leaves


def loss_and_grads(cfg, named, tokens, labels):
    loss, leaves = forward(cfg, named, tokens, labels)
    loss.backward()
    return float(loss), {k: t.grad for k, t in leaves.items()}
