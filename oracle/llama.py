"""PyTorch fp32 Llama forward -- the logits tolerance oracle (TEST ORACLE / CPU BASELINE ONLY).

The reference has no neural model, so the logits oracle is a
plain PyTorch restatement of the architecture the B200 kernels implement
(paper_2408_11850_b200/csrc/llama.cu), over the SAME weight tensors:

  RMSNorm (fp32, x rounded to bf16) -> QKV -> interleaved-pair RoPE -> K/V
  rounded to bf16 -> causal softmax attention (fp32) -> O (+residual) ->
  RMSNorm -> gate/up (rows interleaved) -> SwiGLU (rounded to bf16) -> down
  (+residual) -> final RMSNorm -> lm_head (fp32 logits).

``bf16_points=True`` rounds at exactly the points the kernels store bf16
(activations fed to GEMMs, q/k/v, attention output), so only fp32
accumulation order differs from the GPU; ``bf16_points=False`` is the pure
fp32 math.  ``norm_fold`` selects where RMSNorm's two factors meet the
bf16 rounding, as in the two GEMM engines (paper_2408_11850_b200/csrc/llama.cu):

  norm_fold=False (CUDA-core K2):  y = W . bf16(h * rs * g)
  norm_fold=True  (tcgen05 K3):    y = rs * (W . bf16(h * g))

with rs = 1 / sqrt(mean(h^2) + eps); the two are the same real-number
function of h (and identical when bf16_points=False).  ``OracleLlama`` adds a KV cache and an LCP-reusing ``next_dist``
so the oracle engine (oracle/engine.py) can drive it as the CPU baseline.
"""

from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np
import torch

from .probdist import logits_to_p1, normalize


def _bf(x: torch.Tensor, on: bool) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32) if on else x


def _scaled_inv_freq(inv: np.ndarray, scaling) -> np.ndarray:
    """Hugging Face's rope_scaling rules, branch by branch (linear: every
    frequency / factor; llama3: low band / factor, high band kept, the middle
    band interpolated in original_context / wavelength)."""
    if scaling is None:
        return inv
    if scaling[0] == "linear":
        return inv / scaling[1]
    _, factor, lo, hi, ctx = scaling
    out = inv.copy()
    for i, f in enumerate(inv):
        wl = 2 * math.pi / f
        if wl > ctx / lo:
            out[i] = f / factor
        elif wl >= ctx / hi:
            s = (ctx / wl - lo) / (hi - lo)
            out[i] = (1 - s) * f / factor + s * f
    return out


def rope_tables(hd: int, max_seq: int, theta: float, scaling=None):
    inv = _scaled_inv_freq(theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd), scaling)
    ang = np.arange(max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return torch.from_numpy(np.cos(ang).astype(np.float32)), torch.from_numpy(np.sin(ang).astype(np.float32))


class OracleLlama:
    """fp32 forward over given weights; ``device``/``dtype`` select where it runs.

    ``mm_dtype`` is the matmul operand dtype (float32 for the tolerance
    oracle; bfloat16 makes the CPU baseline practical for 7B-class weights).
    """

    def __init__(self, cfg, weights: Dict, device="cpu", bf16_points: bool = True, max_seq: int = 1024,
                 mm_dtype=torch.float32, bos_id: int = 1, temperature: float = 1.0, norm_fold: bool = False):
        self.cfg = cfg
        self.fold = norm_fold
        self.dev = torch.device(device)
        self.b = bf16_points
        self.mm = mm_dtype
        self.bos_id = bos_id
        self.temperature = temperature
        self.vocab_size = cfg.vocab

        def mv(t):
            return t.to(self.dev).to(mm_dtype if t.dtype == torch.bfloat16 else torch.float32)

        self.embed = weights["embed"].to(self.dev)
        self.lm_head = mv(weights["lm_head"])
        self.final_norm = weights["final_norm"].to(self.dev).float()
        self.layers = [{k: mv(v) for k, v in L.items()} for L in weights["layers"]]
        self.cos, self.sin = rope_tables(cfg.head_dim, max_seq, cfg.rope_theta, getattr(cfg, "rope_scaling", None))
        self.cos, self.sin = self.cos.to(self.dev), self.sin.to(self.dev)
        L, KV, hd = cfg.n_layers, cfg.n_kv_heads, cfg.head_dim
        self.kc = torch.zeros(L, max_seq, KV, hd, device=self.dev)
        self.vc = torch.zeros(L, max_seq, KV, hd, device=self.dev)
        self.cached: List[int] = []

    def _norm(self, h, g):
        """(GEMM operand, per-row scale applied to the GEMM output)."""
        ms = (h * h).mean(dim=-1, keepdim=True)
        rs = torch.rsqrt(ms + self.cfg.norm_eps)
        if self.fold:
            return _bf(h * g, self.b), rs
        return _bf(h * rs * g, self.b), None

    def _mm(self, x, w, scale=None):
        y = (x.to(self.mm) @ w.T).float()
        return y if scale is None else y * scale

    def _rope(self, x, pos):  # x [M, heads, hd]
        c = self.cos[pos][:, None, :]
        s = self.sin[pos][:, None, :]
        a, b = x[..., 0::2], x[..., 1::2]
        out = torch.empty_like(x)
        out[..., 0::2] = a * c - b * s
        out[..., 1::2] = a * s + b * c
        return out

    @torch.no_grad()
    def forward(self, tokens: Sequence[int], start: int) -> torch.Tensor:
        """Logits [M, V] of tokens at positions start.. (cache rows < start reused)."""
        cfg = self.cfg
        M = len(tokens)
        H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        pos = torch.arange(start, start + M, device=self.dev)
        h = self.embed[torch.tensor(list(tokens), device=self.dev)].float()
        for l, Lw in enumerate(self.layers):
            x, rs = self._norm(h, Lw["attn_norm"])
            qkv = self._mm(x, Lw["wqkv"], rs)
            q = qkv[:, :H * hd].view(M, H, hd)
            k = qkv[:, H * hd:(H + KV) * hd].view(M, KV, hd)
            v = qkv[:, (H + KV) * hd:].view(M, KV, hd)
            q = _bf(self._rope(q, pos), self.b)
            k = _bf(self._rope(k, pos), self.b)
            v = _bf(v, self.b)
            self.kc[l, start:start + M] = k
            self.vc[l, start:start + M] = v
            ctx = start + M
            K = self.kc[l, :ctx]  # [ctx, KV, hd]
            Vv = self.vc[l, :ctx]
            rep = H // KV
            K = K.repeat_interleave(rep, dim=1)
            Vv = Vv.repeat_interleave(rep, dim=1)
            s = torch.einsum("mhd,chd->hmc", q, K) / math.sqrt(hd)
            mask = torch.arange(ctx, device=self.dev)[None, :] > pos[:, None]
            s = s.masked_fill(mask[None], float("-inf"))
            p = torch.softmax(s, dim=-1)
            o = _bf(torch.einsum("hmc,chd->mhd", p, Vv).reshape(M, H * hd), self.b)
            h = h + self._mm(o, Lw["wo"])
            x, rs = self._norm(h, Lw["mlp_norm"])
            gu = self._mm(x, Lw["w_gate_up"], rs)
            g, u = gu[:, 0::2], gu[:, 1::2]
            a = _bf(g / (1.0 + torch.exp(-g)) * u, self.b)
            h = h + self._mm(a, Lw["w_down"])
        x, rs = self._norm(h, self.final_norm)
        return self._mm(x, self.lm_head, rs)

    # -- SequenceModel-style adapter for the oracle engine --------------------
    def next_dist(self, prefix: Sequence[int]):
        seq = [self.bos_id] + [int(t) for t in prefix]
        lcp = 0
        lim = min(len(self.cached), len(seq) - 1)
        while lcp < lim and self.cached[lcp] == seq[lcp]:
            lcp += 1
        logits = self.forward(seq[lcp:], lcp)[-1]
        self.cached = seq
        p1 = logits_to_p1(logits.cpu().numpy().astype(np.float32), float(np.float32(1.0 / self.temperature)))

        class _D:
            pass

        d = _D()
        d.probs, _ = normalize(p1)
        return d
