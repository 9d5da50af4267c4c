"""Independent fp64 PyTorch restatement of the BASELINE workloads — TEST
INFRASTRUCTURE ONLY (a second checker beside the oracle for batch sizes the
per-sample oracle cannot finish in seconds).

It restates, with dense torch ops and autograd instead of a scalar tape, the
compositions of csrc/host/tg_models.hpp (the same graphs the reference records
in oracle/_ref): parameter blocks in creation order (make_params), the per-
sample loss of build_sample, and grad_sum = sum_i d f_i / d params
(SPEC.md:431-439 GradAccumulator; backprop.hpp:139-184 per sample).  The
stop-gradient max shift of softmax_ce cancels in the loss and
in its gradient, so plain log-sum-exp is the same function.  Layer norm is the
composed one of SPEC.md:288-296: var = mean(x^2) - mean(x)^2 (biased),
rstd = invSqrt(var + eps).

tests/test_torch_ref.py pins it against the oracle (fp64 tape, the reference
algorithm) to 1e-12 at small batches before the GPU tests trust it at the
BASELINE batch sizes.
"""
from __future__ import annotations

import numpy as np
import torch

DEFAULT_DIMS = {
    "moons": [16, 16],
    "char_mlp": [27, 3, 10, 200],
    "gpt": [65, 64, 64, 4, 4, 256],
    "wide_mlp": [784, 1024, 1024, 10],
}


def resolve(model: str, dims) -> list[int]:
    d = list(DEFAULT_DIMS[model])
    for i, v in enumerate(dims or []):
        if v:
            d[i] = v
    return d


def block_shapes(model: str, dims) -> list[tuple[int, int]]:
    """(rows, cols) of every parameter block in creation order (make_params)."""
    D = resolve(model, dims)
    if model == "moons":
        h1, h2 = D[0], D[1]
        return [(h1, 2), (1, h1), (h2, h1), (1, h2), (1, h2), (1, 1)]
    if model == "char_mlp":
        V, C, E, H = D[:4]
        return [(V, E), (H, C * E), (1, H), (V, H), (1, V)]
    if model == "wide_mlp":
        I, H1, H2, O = D[:4]
        return [(H1, I), (1, H1), (H2, H1), (1, H2), (O, H2), (1, O)]
    if model == "gpt":
        V, T, d, _, L, F = D[:6]
        s = [(V, d), (T, d)]
        for _ in range(L):
            s += [(1, d), (1, d), (3 * d, d), (1, 3 * d), (d, d), (1, d), (1, d), (1, d), (F, d), (1, F), (d, F), (1, d)]
        return s + [(1, d), (1, d), (V, d), (1, V)]
    raise ValueError(model)


def split_params(model: str, dims, flat: torch.Tensor) -> list[torch.Tensor]:
    out, o = [], 0
    for r, c in block_shapes(model, dims):
        out.append(flat[o:o + r * c].view(r, c))
        o += r * c
    assert o == flat.numel(), (o, flat.numel())
    return out


def _ce(z: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    """softmax_ce: log(sum_j exp(z_j - m)) - (z_t - m), per row."""
    return torch.logsumexp(z, dim=-1) - z.gather(-1, target.long().unsqueeze(-1)).squeeze(-1)


def _layer_norm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor, eps: float = 1e-5) -> torch.Tensor:
    mu = x.mean(-1, keepdim=True)
    ms = (x * x).mean(-1, keepdim=True)
    rstd = 1.0 / torch.sqrt(ms - mu * mu + eps)
    return (x - mu) * rstd * g + b


def losses(model: str, dims, P: list[torch.Tensor], x: torch.Tensor | None, k: torch.Tensor | None) -> torch.Tensor:
    """Per-sample losses f_i of build_sample; x: [n_inputs][b], k: [n_index][b]."""
    D = resolve(model, dims)
    if model == "moons":
        W1, b1, W2, b2, W3, b3 = P
        xs = x[:2].t()
        h1 = torch.tanh(xs @ W1.t() + b1[0])
        h2 = torch.tanh(h1 @ W2.t() + b2[0])
        s = h2 @ W3[0] + b3[0, 0]
        reg = 1e-4 * sum((p * p).sum() for p in P)
        return torch.relu(1.0 - x[2] * s) + reg
    if model == "char_mlp":
        V, C, E, H = D[:4]
        emb, W1, b1, W2, b2 = P
        xs = torch.cat([emb[k[c].long()] for c in range(C)], dim=1)       # [b][C*E]
        h = torch.tanh(xs @ W1.t() + b1[0])
        z = h @ W2.t() + b2[0]
        return _ce(z, k[C])
    if model == "wide_mlp":
        W1, b1, W2, b2, W3, b3 = P
        h1 = torch.relu(x.t() @ W1.t() + b1[0])
        h2 = torch.relu(h1 @ W2.t() + b2[0])
        z = h2 @ W3.t() + b3[0]
        return _ce(z, k[0])
    if model == "gpt":
        V, T, d, H, L, F = D[:6]
        hd = d // H
        wte, wpe = P[0], P[1]
        tok = k[:T].t().long()                                             # [b][T]
        h = wte[tok] + wpe[:T]                                             # [b][T][d]
        scale = 1.0 / np.sqrt(hd)
        mask = torch.ones(T, T, dtype=torch.bool, device=h.device).tril()
        for l in range(L):
            g1, be1, Wqkv, bqkv, Wo, bo, g2, be2, W1, b1, W2, b2 = P[2 + 12 * l: 14 + 12 * l]
            qkv = _layer_norm(h, g1[0], be1[0]) @ Wqkv.t() + bqkv[0]       # [b][T][3d]
            bsz = qkv.shape[0]
            q, kk, v = (qkv[..., i * d:(i + 1) * d].view(bsz, T, H, hd).transpose(1, 2) for i in range(3))
            sc = (q @ kk.transpose(-1, -2)) * scale
            sc = sc.masked_fill(~mask, float("-inf"))
            a = torch.softmax(sc, dim=-1)
            att = (a @ v).transpose(1, 2).reshape(bsz, T, d)
            h = h + (att @ Wo.t() + bo[0])
            f1 = torch.relu(_layer_norm(h, g2[0], be2[0]) @ W1.t() + b1[0])
            h = h + (f1 @ W2.t() + b2[0])
        o = 2 + 12 * L
        z = _layer_norm(h, P[o][0], P[o + 1][0]) @ P[o + 2].t() + P[o + 3][0]   # [b][T][V]
        return _ce(z, k[1:T + 1].t()).mean(dim=1)
    raise ValueError(model)


def run(model: str, dims, params, x, k, device="cpu", chunk: int = 0, dtype=torch.float64) -> dict:
    """Losses [b] and grad_sum [n_params] as float64 numpy (chunked over
    samples).  dtype float32 gives an independent fp32 implementation (plain
    fp32 matmuls, TF32 off) whose own distance from the fp64 result measures
    how far fp32 arithmetic alone moves the gradient at a batch size."""
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    flat = torch.tensor(np.asarray(params, np.float64), device=device, dtype=dtype, requires_grad=True)
    Xt = torch.as_tensor(np.asarray(x)) if x is not None and np.asarray(x).size else None
    Kt = torch.as_tensor(np.asarray(k, np.int32)) if k is not None and np.asarray(k).size else None
    b = (Xt.shape[1] if Xt is not None else Kt.shape[1])
    chunk = chunk or b
    out = np.zeros(b)
    for lo in range(0, b, chunk):
        hi = min(b, lo + chunk)
        xs = Xt[:, lo:hi].to(device, dtype) if Xt is not None else None
        ks = Kt[:, lo:hi].to(device) if Kt is not None else None
        P = split_params(model, dims, flat)
        f = losses(model, dims, P, xs, ks)
        f.sum().backward()
        out[lo:hi] = f.detach().cpu().numpy()
    return {"loss": out, "grad_sum": flat.grad.detach().cpu().double().numpy()}
