"""GPU Llama SequenceModels: random-init weights of the named architectures.

``LlamaModel`` is a ``SequenceModel`` (its ``next_dist`` is an adapter over
the device forward, for the plugin path and for parity runs of the
reference engine) and a *device model*: the engines' fast path drives its
KV-cached forward (libpearl_b200 ``pearl_llama_forward``) directly.

Architectures (public model-card values; PAPER.md:571-580 gives L/d/FFN,
heads / KV heads / vocab are external):

    llama2-7b    L32 d4096 H32/32 FFN11008 V32000      (target, C2)
    llama-68m    L2  d768  H12/12 FFN3072  V32000      (draft,  C2)
    dsc-33b      L62 d7168 H56/8  FFN19200 V32256      (target, C3)
    dsc-1.3b     L24 d2048 H16/16 FFN5504  V32256      (draft,  C3)
    llama3-70b   L80 d8192 H64/8  FFN28672 V128256     (target, C4)
    llama3-8b    L32 d4096 H32/8  FFN14336 V128256     (draft,  C4)
    tiny-target  L4  d512  H8/8   FFN1376  V32000      (C1, builder-defined)
    tiny-draft   L2  d256  H4/4   FFN688   V32000      (C1)

Controlled-alignment random init (no checkpoints exist offline; random
independent pairs would accept ~0 drafts at T=0): both models of a pair share
a rank-r bigram structure -- embeddings E = sqrt(d) * U_hat P and lm_head =
kappa * U'_hat P / sqrt(d), with P an orthonormal r x d projection drawn per
model, U_hat a shared random unit-row table and U' = U_hat permuted (token
x's successor pi(x) scores kappa).  Every other weight is i.i.d. Gaussian
(std 0.02; attention-out and MLP-down use ``branch_std``), so each model's
context-dependent residual branches perturb the shared bigram law
independently; ``branch_std`` is the alignment knob and the measured
acceptance is always reported next to any speedup.
"""

from __future__ import annotations

import ctypes
import os
import math
import time
from dataclasses import dataclass, replace
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _device, _lib
from .core import ProbDist
from .models import LatencyProfile, SequenceModel


@dataclass(frozen=True)
class LlamaConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    # ("linear", factor) or ("llama3", factor, low_freq_factor, high_freq_factor,
    # original_max_position_embeddings); None = plain RoPE (checkpoint.config_from_hf)
    rope_scaling: Optional[tuple] = None
    bos_id: int = 1
    eos_id: Optional[int] = None

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def param_count(self) -> int:
        d, hd = self.d_model, self.head_dim
        per_layer = d * (self.n_heads + 2 * self.n_kv_heads) * hd + self.n_heads * hd * d + 3 * d * self.ffn + 2 * d
        return self.n_layers * per_layer + 2 * self.vocab * d + d

    def weight_bytes(self) -> int:
        """bf16 bytes streamed per forward (norms are fp32 here but tiny)."""
        d, hd = self.d_model, self.head_dim
        mats = self.n_layers * (d * (self.n_heads + 2 * self.n_kv_heads) * hd + self.n_heads * hd * d
                                + 3 * d * self.ffn) + self.vocab * d
        return 2 * mats

    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2


PRESETS: Dict[str, LlamaConfig] = {
    "llama2-7b": LlamaConfig("llama2-7b", 32, 4096, 32, 32, 11008, 32000),
    "llama-68m": LlamaConfig("llama-68m", 2, 768, 12, 12, 3072, 32000),
    "dsc-33b": LlamaConfig("dsc-33b", 62, 7168, 56, 8, 19200, 32256, rope_theta=100000.0, norm_eps=1e-6),
    "dsc-1.3b": LlamaConfig("dsc-1.3b", 24, 2048, 16, 16, 5504, 32256, rope_theta=100000.0, norm_eps=1e-6),
    "llama3-70b": LlamaConfig("llama3-70b", 80, 8192, 64, 8, 28672, 128256, rope_theta=500000.0),
    "llama3-8b": LlamaConfig("llama3-8b", 32, 4096, 32, 8, 14336, 128256, rope_theta=500000.0),
    "tiny-target": LlamaConfig("tiny-target", 4, 512, 8, 8, 1376, 32000),
    "tiny-draft": LlamaConfig("tiny-draft", 2, 256, 4, 4, 688, 32000),
}

PAIRS = {
    "tiny": ("tiny-target", "tiny-draft"),
    "llama2-7b/68m": ("llama2-7b", "llama-68m"),
    "dsc-33b/1.3b": ("dsc-33b", "dsc-1.3b"),
    "llama3-70b/8b": ("llama3-70b", "llama3-8b"),
}


# alignment knob per pair, calibrated on B200 to alpha-hat ~0.9 at T=1 (tools/calib_alpha.py)
PAIR_BRANCH_STD = {"llama2-7b/68m": 5e-4, "dsc-33b/1.3b": 1.7e-4, "llama3-70b/8b": 8e-5, "tiny": 2e-4}
# SMs of the green-context partition PEARL's concurrent draft runs on (the
# target keeps the rest; 0 = shared SMs; the driver rounds to 8-SM groups).  On
# its own SMs the 68M draft stops competing with the target's GEMM CTAs for SM
# slots, and enough of them let it keep up with long draft blocks.  Round-2
# sweep with the round-2 kernels (tools/gpu_draftsms.sh, T=1, live planner
# calibration): PEARL 1158 / 1372 / 1378 / 1451 / 1341 tok/s at 16 / 24 / 32 /
# 40 / 48 SMs; session 3, with the single-token GEMV (tools/_r2s3_draftsms.sh):
# 1529 / 1761 / 1455 / 1473 tok/s at 24 / 32 / 40 / 48 SMs on 5 prompts, which is
# noise: on 20 prompts 1332 / 1337 / 1334 / 1260 (profiles/r02_s3/draftsms20_*.json).
# DSC-33B/1.3B (prompt 512): 48 SMs (round 1: shared 130 tok/s, 48
# SMs 163).  Llama-3 (V = 128256) needs 16-CTA clusters for its pick / verify,
# which a partition cannot host: shared SMs.
PAIR_DRAFT_SMS = {"llama2-7b/68m": 32, "dsc-33b/1.3b": 48, "llama3-70b/8b": 0, "tiny": 0}


@dataclass(frozen=True)
class AlignSpec:
    """Controlled-alignment knobs of a random-init pair (see module doc)."""

    rank: int = 64
    kappa: float = 13.0
    branch_std: float = 2e-4
    seed: int = 1234


def rope_inv_freq(hd: int, theta: float, scaling: Optional[tuple] = None) -> np.ndarray:
    """RoPE inverse frequencies (fp64), with the checkpoint's ``rope_scaling``:
    "linear" divides every frequency by the factor (positions / factor);
    "llama3" divides the low frequencies (wavelength > original context /
    low_freq_factor) by the factor, keeps the high ones (wavelength < original
    context / high_freq_factor) and interpolates linearly in
    original_context / wavelength between them."""
    inv = theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    if scaling is None:
        return inv
    if scaling[0] == "linear":
        return inv / float(scaling[1])
    if scaling[0] == "llama3":
        _, factor, lo, hi, ctx = scaling
        wavelen = 2.0 * math.pi / inv
        mix = np.clip((ctx / wavelen - lo) / (hi - lo), 0.0, 1.0)  # 0: scaled, 1: kept
        return (1.0 - mix) * inv / factor + mix * inv
    raise ValueError(f"unsupported rope scaling {scaling[0]!r}")


def rope_tables(hd: int, max_seq: int, theta: float, scaling: Optional[tuple] = None):
    inv = rope_inv_freq(hd, theta, scaling)
    ang = np.arange(max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def _shared_tables(V: int, align: AlignSpec, device) -> tuple:
    g = torch.Generator(device=device)
    g.manual_seed(align.seed)
    U = torch.randn(V, align.rank, generator=g, device=device, dtype=torch.float32)
    U = U / U.norm(dim=1, keepdim=True)
    perm = torch.randperm(V, generator=g, device=device)
    Uo = torch.empty_like(U)
    Uo[perm] = U  # successor of token x is perm[x]: its output vector is U[x]
    Uo = Uo + 0.05 * torch.randn(V, align.rank, generator=g, device=device) / math.sqrt(align.rank)
    return U, Uo


def init_weights(cfg: LlamaConfig, align: AlignSpec, model_seed: int, device,
                 shared=None) -> Dict[str, object]:
    """Random-init weights (bf16 matrices, fp32 norms) with the shared bigram structure."""
    g = torch.Generator(device=device)
    g.manual_seed(model_seed)
    d, hd, H, KV, F, V = cfg.d_model, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.vocab
    U, Uo = shared if shared is not None else _shared_tables(V, align, device)
    q, _ = torch.linalg.qr(torch.randn(d, align.rank, generator=g, device=device, dtype=torch.float32))
    P = q.T.contiguous()  # r x d, orthonormal rows
    w: Dict[str, object] = {}
    emb = torch.empty(V, d, dtype=torch.bfloat16, device=device)
    head = torch.empty(V, d, dtype=torch.bfloat16, device=device)
    for s in range(0, V, 16384):
        emb[s:s + 16384] = (math.sqrt(d) * (U[s:s + 16384] @ P)).to(torch.bfloat16)
        head[s:s + 16384] = (align.kappa / math.sqrt(d) * (Uo[s:s + 16384] @ P)).to(torch.bfloat16)
    w["embed"], w["lm_head"] = emb, head
    w["final_norm"] = torch.ones(d, dtype=torch.float32, device=device)

    def rnd(rows, cols, std):
        t = torch.empty(rows, cols, dtype=torch.bfloat16, device=device)
        for s in range(0, rows, 4096):
            e = min(rows, s + 4096)
            t[s:e] = (torch.randn(e - s, cols, generator=g, device=device) * std).to(torch.bfloat16)
        return t

    layers = []
    for _ in range(cfg.n_layers):
        layers.append({
            "attn_norm": torch.ones(d, dtype=torch.float32, device=device),
            "wqkv": rnd((H + 2 * KV) * hd, d, 0.02),
            "wo": rnd(d, H * hd, align.branch_std),
            "mlp_norm": torch.ones(d, dtype=torch.float32, device=device),
            "w_gate_up": rnd(2 * F, d, 0.02),  # rows 2j = gate_j, 2j+1 = up_j
            "w_down": rnd(d, F, align.branch_std),
        })
    w["layers"] = layers
    return w


def pair_configs(pair: str, depth: Optional[tuple] = None) -> tuple:
    """(target_cfg, draft_cfg) of a named pair; ``depth=(Lt, Ld)`` keeps every
    width (d, heads, KV heads, FFN, vocab, rope theta) and only cuts the layer
    count -- the reduced-depth, full-width parity configs."""
    tname, dname = PAIRS[pair]
    tc, dc = PRESETS[tname], PRESETS[dname]
    if depth is not None:
        tc = replace(tc, name=f"{tc.name}-L{depth[0]}", n_layers=int(depth[0]))
        dc = replace(dc, name=f"{dc.name}-L{depth[1]}", n_layers=int(depth[1]))
    return tc, dc


def init_pair(pair: str, align: AlignSpec = AlignSpec(), device=None, depth: Optional[tuple] = None):
    """(target_weights, draft_weights, target_cfg, draft_cfg) for a named pair."""
    device = device or _device.require_cuda()
    tc, dc = pair_configs(pair, depth)
    assert tc.vocab == dc.vocab
    shared = _shared_tables(tc.vocab, align, device)
    tw = init_weights(tc, align, align.seed + 1, device, shared)
    dw = init_weights(dc, align, align.seed + 2, device, shared)
    del shared
    return tw, dw, tc, dc


class _CConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "ffn",
                                              "vocab", "max_seq", "max_tokens", "gemm_kind")] + [
        ("norm_eps", ctypes.c_float), ("sm_count", ctypes.c_int32), ("n_slots", ctypes.c_int32)]


GEMM_KINDS = {"cudacore": 0, "tcgen05": 1}


def _pack_streamed(w: Dict[str, object]):
    """Copy every per-token streamed tensor (lm_head, final norm, all layer
    weights; not the embedding table, which is only gathered) into one
    contiguous device buffer and point ``w`` at views of it."""
    items = [(w, "lm_head"), (w, "final_norm")]
    for L in w["layers"]:
        items += [(L, k) for k in ("attn_norm", "wqkv", "wo", "mlp_norm", "w_gate_up", "w_down")]
    offs, total = [], 0
    for d, k in items:
        offs.append(total)
        total += (d[k].numel() * d[k].element_size() + 255) // 256 * 256
    buf = torch.empty(total, dtype=torch.uint8, device=w["lm_head"].device)
    for (d, k), off in zip(items, offs):
        t = d[k]
        v = buf[off:off + t.numel() * t.element_size()].view(t.dtype).view(t.shape)
        v.copy_(t)
        d[k] = v
    return buf, total


class LlamaModel(SequenceModel):
    """A random-init Llama on the GPU: SequenceModel + device fast-path model."""

    _pearl_device_model = True

    def __init__(self, cfg: LlamaConfig, weights: Dict[str, object], gemm: str = "cudacore",
                 max_seq: int = 1024, max_tokens: int = 64, temperature: float = 1.0, bos_id: Optional[int] = None,
                 latency: Optional[LatencyProfile] = None, l2_resident: bool = False, sm_count: int = 0,
                 n_slots: int = 1):
        self.device = _device.require_cuda()
        self.cfg = cfg
        self.vocab_size = cfg.vocab
        self.temperature = float(temperature)
        self.bos_id = int(cfg.bos_id if bos_id is None else bos_id)
        self.max_seq = int(max_seq)
        self.max_tokens = int(max_tokens)
        self.gemm = gemm
        self.w = weights
        # streamed weights packed contiguously so one L2 access-policy window covers them
        self._l2_pack = _pack_streamed(weights) if l2_resident else None
        hd = cfg.head_dim
        cos, sin = rope_tables(hd, max_seq, cfg.rope_theta, cfg.rope_scaling)
        self.rope_cos = torch.from_numpy(cos).to(self.device)
        self.rope_sin = torch.from_numpy(sin).to(self.device)
        # KV cache [L, slots, max_seq, KV, hd]: slot 0 serves the single-sequence
        # engines, slots 0..n_slots-1 the batched ones (batched.py)
        self.n_slots = int(n_slots)
        kv_shape = (cfg.n_layers, self.n_slots, max_seq, cfg.n_kv_heads, hd)
        self.k_cache = torch.zeros(kv_shape, dtype=torch.bfloat16, device=self.device)
        self.v_cache = torch.zeros(kv_shape, dtype=torch.bfloat16, device=self.device)
        ptrs = [weights["embed"], weights["final_norm"], weights["lm_head"], self.rope_cos, self.rope_sin,
                self.k_cache, self.v_cache]
        for L in weights["layers"]:
            ptrs += [L["attn_norm"], L["wqkv"], L["wo"], L["mlp_norm"], L["w_gate_up"], L["w_down"]]
        for t in ptrs:
            assert t.is_cuda and t.is_contiguous()
        self._ptr_arr = (ctypes.c_void_p * len(ptrs))(*[t.data_ptr() for t in ptrs])
        c = _CConfig(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, hd, cfg.ffn, cfg.vocab, max_seq,
                     max_tokens, GEMM_KINDS[gemm], cfg.norm_eps, int(sm_count), self.n_slots)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pearl_llama_create(ctypes.byref(c), self._ptr_arr, len(ptrs), ctypes.byref(h)),
                   "pearl_llama_create")
        self.handle = h
        self.l2_granted = 0
        if self._l2_pack is not None:
            buf, nbytes = self._l2_pack
            granted = ctypes.c_size_t(0)
            _lib.check(_lib.load().pearl_llama_set_l2_window(h, buf.data_ptr(), nbytes, ctypes.byref(granted)),
                       "pearl_llama_set_l2_window")
            self.l2_granted = int(granted.value)
        _lib.prepare_vocab(cfg.vocab)
        # adapter state (next_dist): tokens whose K/V occupy cache positions 0..n-1
        self._pos = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._cached: List[int] = []
        self._latency = latency

    # -- device API -------------------------------------------------------
    def forward(self, tokens: torch.Tensor, n: int, pos: torch.Tensor, flags: int, logits: Optional[torch.Tensor],
                stream=None) -> None:
        _lib.check(_lib.load().pearl_llama_forward(self.handle, _device.ptr(tokens), int(n), _device.ptr(pos),
                                                   int(flags), _device.ptr(logits), _device.stream_ptr(stream)),
                   "pearl_llama_forward")

    def forward_slots(self, tokens: torch.Tensor, n: int, tok_slot: torch.Tensor, tok_pos: torch.Tensor,
                      logits: Optional[torch.Tensor], stream=None) -> None:
        """Batched forward: token i at position tok_pos[i] of KV slot tok_slot[i] (device int32)."""
        _lib.check(_lib.load().pearl_llama_forward_slots(self.handle, _device.ptr(tokens), int(n), _device.ptr(tok_slot),
                                                         _device.ptr(tok_pos), _device.ptr(logits),
                                                         _device.stream_ptr(stream)), "pearl_llama_forward_slots")

    def forward_logits(self, tokens: Sequence[int], start: int = 0) -> torch.Tensor:
        """fp32 logits of every token of ``tokens`` placed at positions start.. (fresh cache)."""
        toks = torch.tensor(list(tokens), dtype=torch.int32, device=self.device)
        pos = torch.tensor([start], dtype=torch.int32, device=self.device)
        out = torch.empty(len(tokens), self.cfg.vocab, dtype=torch.float32, device=self.device)
        T = self.max_tokens
        for s in range(0, len(tokens), T):
            n = min(T, len(tokens) - s)
            self.forward(toks[s:s + n], n, pos, 1, out[s:s + n])
        self._cached = []  # cache content no longer tracks the adapter
        return out

    @property
    def latency(self) -> LatencyProfile:
        if self._latency is None:
            self._latency = LatencyProfile(self.measure_forward_time(1))
        return self._latency

    @latency.setter
    def latency(self, v: LatencyProfile) -> None:
        self._latency = v

    def measure_forward_time(self, n_tokens: int = 1, iters: int = 5) -> float:
        """Measured seconds per forward of an n-token window (CUDA events)."""
        toks = torch.full((n_tokens,), self.bos_id, dtype=torch.int32, device=self.device)
        pos = torch.zeros(1, dtype=torch.int32, device=self.device)
        out = torch.empty(n_tokens, self.cfg.vocab, dtype=torch.float32, device=self.device)
        for _ in range(2):
            self.forward(toks, n_tokens, pos, 0, out)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            self.forward(toks, n_tokens, pos, 0, out)
        e.record()
        e.synchronize()
        self._cached = []
        return s.elapsed_time(e) / 1e3 / iters

    # -- SequenceModel adapter ---------------------------------------------
    def next_dist(self, prefix: Sequence[int]) -> ProbDist:
        """ProbDist of the device law after ``prefix`` (LCP-reused KV cache).

        The law is the device softmax p1 of the fp32 logits (the same one the
        fast path's kernels use), handed to ProbDist which renormalises it
        exactly like the reference.
        """
        seq = [self.bos_id] + [int(t) for t in prefix]
        lcp = 0
        lim = min(len(self._cached), len(seq) - 1)
        while lcp < lim and self._cached[lcp] == seq[lcp]:
            lcp += 1
        todo = seq[lcp:]
        if len(seq) > self.max_seq:
            raise ValueError("prefix exceeds the KV-cache capacity")
        self._pos.fill_(lcp)
        toks = torch.tensor(todo, dtype=torch.int32, device=self.device)
        logits = torch.empty(1, self.cfg.vocab, dtype=torch.float32, device=self.device)
        self.forward(toks, len(todo), self._pos, _FWD_LAST, logits)
        self._cached = seq
        return ProbDist(self.probs_from_logits(logits)[0].cpu().numpy())

    def probs_from_logits(self, logits: torch.Tensor, temperature: Optional[float] = None) -> torch.Tensor:
        t = self.temperature if temperature is None else temperature
        n = logits.shape[0]
        out = torch.empty(n, self.cfg.vocab, dtype=torch.float64, device=self.device)
        st = torch.zeros(1, dtype=torch.int32, device=self.device)
        _lib.check(_lib.load().pearl_logits_to_probs(_device.ptr(logits), n, self.cfg.vocab,
                                                     float(np.float32(1.0 / t)), _device.ptr(out),
                                                     _device.ptr(st), _device.stream_ptr()), "logits_to_probs")
        _lib.check(int(st.item()), "logits_to_probs")
        return out

    def reset_adapter(self) -> None:
        self._cached = []

    def clone(self, sm_count: int = 0, n_slots: Optional[int] = None) -> "LlamaModel":
        """A second device model over the SAME weight tensors (no copy) with its
        own KV cache and workspace -- e.g. the target on the whole GPU for AR /
        SD next to the SM-partitioned one PEARL's concurrent step uses."""
        return LlamaModel(self.cfg, self.w, gemm=self.gemm, max_seq=self.max_seq, max_tokens=self.max_tokens,
                          temperature=self.temperature, bos_id=self.bos_id, latency=self._latency,
                          sm_count=sm_count, n_slots=self.n_slots if n_slots is None else n_slots)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _destroy_handle(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# Handles whose release fell inside a CUDA graph capture (a garbage-collected
# model while another model's step graph is being captured): cudaFree is not
# capturable, so they are destroyed at the next release outside a capture.
_PENDING_DESTROY: List[int] = []


def _capturing() -> bool:
    try:
        return torch.cuda.is_available() and torch.cuda.is_current_stream_capturing()
    except Exception:
        return False


def _destroy_handle(handle) -> None:
    if _capturing():
        _PENDING_DESTROY.append(handle)
        return
    lib = _lib.load()
    while _PENDING_DESTROY:
        lib.pearl_llama_destroy(_PENDING_DESTROY.pop())
    lib.pearl_llama_destroy(handle)


_FWD_ADVANCE = 1
_FWD_LAST = 2


def inv_temp(t: float) -> float:
    """fp32 inverse temperature exactly as the kernels receive it."""
    return float(np.float32(1.0 / t))


def build_pair(pair: str = "tiny", gemm_target: str = "cudacore", gemm_draft: str = "auto",
               align: AlignSpec = AlignSpec(), max_seq: int = 1024, max_tokens: int = 64,
               temperature: float = 1.0, l2_draft: Optional[bool] = None, draft_sms: Optional[int] = None,
               n_slots: int = 1, depth: Optional[tuple] = None):
    """(target LlamaModel, draft LlamaModel) with controlled-alignment random weights.

    ``l2_draft``: keep the draft's streamed weights in persisting L2
    (PEARL_L2_DRAFT, default off).  ``draft_sms``: run PEARL's concurrent
    draft on its own partition of that many SMs and the target on the rest
    (green contexts; PEARL_DRAFT_SMS, default 0 = shared SMs).  The target's
    stream-K grids are then sized to its partition for every engine, so AR,
    SD and PEARL stay bitwise consistent.  ``gemm_draft="auto"``: the CUDA-core
    GEMV (K2) for drafts under 1 GB of weights, where a forward is
    launch-latency bound and K2 is as fast; tcgen05 (K3) for larger drafts,
    where it streams faster (tools/draft_times.py: 1.3B 1.21 vs 1.50 ms,
    8B 3.41 vs 4.51 ms per token on B200).  ``depth=(Lt, Ld)``: reduced-depth,
    full-width variant of the pair (parity tests at the BASELINE shapes)."""
    tw, dw, tc, dc = init_pair(pair, align, depth=depth)
    return pair_from_weights(tc, tw, dc, dw, gemm_target=gemm_target, gemm_draft=gemm_draft, max_seq=max_seq,
                             max_tokens=max_tokens, temperature=temperature, l2_draft=l2_draft,
                             draft_sms=draft_sms, n_slots=n_slots)


def pair_from_weights(tc: LlamaConfig, tw, dc: LlamaConfig, dw, gemm_target: str = "cudacore",
                      gemm_draft: str = "auto", max_seq: int = 1024, max_tokens: int = 64,
                      temperature: float = 1.0, l2_draft: Optional[bool] = None,
                      draft_sms: Optional[int] = None, n_slots: int = 1):
    """(target LlamaModel, draft LlamaModel) over given weights (random-init
    pairs and checkpoints alike); the knobs are build_pair's."""
    if l2_draft is None:
        l2_draft = os.environ.get("PEARL_L2_DRAFT", "0") == "1"
    if draft_sms is None:
        draft_sms = int(os.environ.get("PEARL_DRAFT_SMS", "0"))
    green = None
    target_sms = 0
    if draft_sms > 0 and tc.vocab > 65536:
        # the pick / K1 kernels run 16-CTA clusters at V > 65536, which a
        # partition's GPC slices cannot host (cudaErrorInvalidClusterSize)
        import warnings
        warnings.warn("green-context draft partition needs V <= 65536 (8-CTA clusters); using shared SMs")
        draft_sms = 0
    if draft_sms > 0:
        _device.require_cuda()
        ds, ts = ctypes.c_void_p(), ctypes.c_void_p()
        nd, nt = ctypes.c_int(0), ctypes.c_int(0)
        rc = _lib.load().pearl_green_streams(int(draft_sms), ctypes.byref(ds), ctypes.byref(ts), ctypes.byref(nd),
                                             ctypes.byref(nt))
        if rc == 0:
            green = (ds.value, ts.value, nd.value, nt.value)
            target_sms = nt.value
        else:  # no green contexts on this driver / device: shared SMs
            import warnings
            warnings.warn(f"green-context partition unavailable ({_lib.load().pearl_last_error().decode()}); "
                          "draft and target share all SMs")
    target = LlamaModel(tc, tw, gemm=gemm_target, max_seq=max_seq,
                        max_tokens=max_tokens if gemm_target == "tcgen05" else min(max_tokens, 64),
                        temperature=temperature, sm_count=target_sms, n_slots=n_slots)
    if gemm_draft == "auto":
        gemm_draft = "tcgen05" if dc.weight_bytes() > 1e9 else "cudacore"
    # the CUDA-core engine's fused-norm prologue takes <= 64 tokens per pass
    draft_tokens = max_tokens if gemm_draft == "tcgen05" else min(max_tokens, 64)
    # a draft on its own partition sizes its persistent grids to it (tcgen05
    # stream-K grids; the CUDA-core model's single-token persistent forward,
    # whose grid barrier needs every CTA co-resident)
    draft = LlamaModel(dc, dw, gemm=gemm_draft, max_seq=max_seq, max_tokens=draft_tokens, temperature=temperature,
                       l2_resident=l2_draft, n_slots=n_slots, sm_count=green[2] if green is not None else 0)
    if green is not None:
        target.green_partition = green  # (draft stream, target stream, draft SMs, target SMs)
    return target, draft
