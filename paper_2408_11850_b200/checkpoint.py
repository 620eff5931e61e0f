"""Real checkpoints: Hugging Face Llama safetensors -> the B200 weight layout.

The bench runs random-init weights (no network for checkpoints here), but the
runtime takes real ones.  This module reads ``model*.safetensors`` shards (the
format is parsed directly: an 8-byte header length, a JSON header, raw
little-endian tensors) and ``config.json``, and repacks the tensors into the
layout the kernels stream (llama.py / include/pearl_b200.h):

* ``wqkv`` = rows of q_proj, k_proj, v_proj concatenated, with every head's
  rows re-ordered from Hugging Face's rotate-half RoPE layout (row i pairs
  with row i + hd/2) to the adjacent-pair layout the QKV epilogue rotates
  (rows 2i, 2i+1) -- the inverse of the permutation HF's conversion script
  applies to Meta's checkpoints, so the rotated q/k values are identical;
* ``w_gate_up`` = gate_proj / up_proj rows interleaved (2j = gate_j,
  2j+1 = up_j) so SwiGLU fuses into the GEMM epilogue;
* ``wo`` / ``w_down`` / ``embed`` / ``lm_head`` as bf16 matrices (lm_head =
  embed_tokens when the embeddings are tied), RMSNorm gains as fp32.

``load_llama(path)`` returns ``(LlamaConfig, weights)`` ready for
``llama.LlamaModel(cfg, weights, ...)``.
"""

from __future__ import annotations

import glob
import json
import os
import struct
from typing import Dict, Optional, Tuple

import torch

from .llama import LlamaConfig

_DTYPES = {"BF16": (torch.bfloat16, 2), "F16": (torch.float16, 2), "F32": (torch.float32, 4)}


def _header(path: str):
    with open(path, "rb") as fh:
        (n,) = struct.unpack("<Q", fh.read(8))
        return json.loads(fh.read(n)), 8 + n


def _read_tensor(path: str, base: int, name: str, meta: dict) -> torch.Tensor:
    dt = meta["dtype"]
    if dt not in _DTYPES:
        raise ValueError(f"{path}: tensor {name} has unsupported dtype {dt}")
    tdt, _ = _DTYPES[dt]
    lo, hi = meta["data_offsets"]
    with open(path, "rb") as fh:
        fh.seek(base + lo)
        raw = bytearray(fh.read(hi - lo))
    t = torch.frombuffer(raw, dtype=tdt) if raw else torch.empty(0, dtype=tdt)
    return t.reshape(meta["shape"])


def read_safetensors(path: str) -> Dict[str, torch.Tensor]:
    """All tensors of one .safetensors file as CPU torch tensors."""
    header, base = _header(path)
    return {name: _read_tensor(path, base, name, meta) for name, meta in header.items() if name != "__metadata__"}


class LazyShards:
    """name -> tensor over a checkpoint's shards, read from disk on access
    (nothing is cached), so packing holds one layer on the host at a time."""

    def __init__(self, paths):
        self._where = {}
        for path in paths:
            header, base = _header(path)
            for name, meta in header.items():
                if name != "__metadata__":
                    self._where[name] = (path, base, meta)

    def __len__(self):
        return len(self._where)

    def __contains__(self, name):
        return name in self._where

    def __getitem__(self, name) -> torch.Tensor:
        path, base, meta = self._where[name]
        return _read_tensor(path, base, name, meta)

    def get(self, name, default=None):
        return self[name] if name in self._where else default


def write_safetensors(path: str, tensors: Dict[str, torch.Tensor]) -> None:
    """Minimal writer (tests and tooling): contiguous tensors, sorted names."""
    names = sorted(tensors)
    header, blobs, off = {}, [], 0
    rev = {v[0]: k for k, v in _DTYPES.items()}
    for name in names:
        t = tensors[name].contiguous()
        b = t.view(torch.uint8).numpy().tobytes() if t.dtype == torch.bfloat16 else t.numpy().tobytes()
        header[name] = {"dtype": rev[t.dtype], "shape": list(t.shape), "data_offsets": [off, off + len(b)]}
        blobs.append(b)
        off += len(b)
    hj = json.dumps(header).encode()
    hj += b" " * ((8 - len(hj) % 8) % 8)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", len(hj)))
        fh.write(hj)
        for b in blobs:
            fh.write(b)


def _rope_scaling(rs) -> Optional[tuple]:
    """config.json ``rope_scaling`` -> LlamaConfig.rope_scaling (llama.rope_inv_freq).
    Linear (DeepSeek-Coder) and llama3 (Llama-3.1+) are applied; any other
    type (dynamic NTK, yarn, longrope) is rejected rather than silently
    ignored, since it would change the RoPE tables and hence every logit."""
    if not rs:
        return None
    kind = rs.get("rope_type", rs.get("type"))
    if kind in (None, "default"):
        return None
    if kind == "linear":
        return ("linear", float(rs["factor"]))
    if kind == "llama3":
        return ("llama3", float(rs["factor"]), float(rs["low_freq_factor"]), float(rs["high_freq_factor"]),
                float(rs["original_max_position_embeddings"]))
    raise ValueError(f"unsupported rope_scaling type {kind!r} (supported: linear, llama3)")


def _first_id(v) -> Optional[int]:
    """bos/eos ids may be an int, a list (Llama-3.1 lists several EOS ids; the
    engines stop at one: the first) or null."""
    if isinstance(v, (list, tuple)):
        v = v[0] if v else None
    return None if v is None else int(v)


def config_from_hf(cfg: dict, name: str = "hf-llama") -> LlamaConfig:
    """LlamaConfig from a Hugging Face config.json (LlamaForCausalLM),
    including rope_scaling and the BOS / EOS token ids."""
    H = int(cfg["num_attention_heads"])
    d = int(cfg["hidden_size"])
    hd = int(cfg.get("head_dim", d // H))
    if hd * H != d:
        raise ValueError("head_dim * num_attention_heads must equal hidden_size")
    V = int(cfg["vocab_size"])
    if V % 4:
        raise ValueError(f"vocab_size {V} is not a multiple of 4: the kernels stream 16-byte aligned logits rows")
    bos = _first_id(cfg.get("bos_token_id"))
    return LlamaConfig(name, int(cfg["num_hidden_layers"]), d, H, int(cfg.get("num_key_value_heads", H)),
                       int(cfg["intermediate_size"]), V,
                       rope_theta=float(cfg.get("rope_theta", 10000.0)), norm_eps=float(cfg.get("rms_norm_eps", 1e-5)),
                       rope_scaling=_rope_scaling(cfg.get("rope_scaling")),
                       bos_id=1 if bos is None else bos, eos_id=_first_id(cfg.get("eos_token_id")))


def rotate_half_to_adjacent(w: torch.Tensor, n_heads: int, hd: int) -> torch.Tensor:
    """Re-order each head's rows from rotate-half pairs (i, i + hd/2) to
    adjacent pairs (2i, 2i + 1)."""
    rows = w.shape[1]
    return w.reshape(n_heads, 2, hd // 2, rows).transpose(1, 2).reshape(n_heads * hd, rows)


def pack_hf_llama(t: Dict[str, torch.Tensor], cfg: LlamaConfig, device=None) -> Dict[str, object]:
    """Repack HF tensor names into the kernels' layout (see module doc)."""
    dev = device or "cpu"
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim

    def bf(x):
        return x.to(torch.bfloat16).contiguous().to(dev)

    def f32(x):
        return x.to(torch.float32).contiguous().to(dev)

    p = "model."
    emb = bf(t[p + "embed_tokens.weight"])
    w: Dict[str, object] = {"embed": emb, "lm_head": bf(t["lm_head.weight"]) if "lm_head.weight" in t else emb,
                            "final_norm": f32(t[p + "norm.weight"])}
    layers = []
    for i in range(cfg.n_layers):
        q = f"{p}layers.{i}."
        wq = rotate_half_to_adjacent(t[q + "self_attn.q_proj.weight"], H, hd)
        wk = rotate_half_to_adjacent(t[q + "self_attn.k_proj.weight"], KV, hd)
        wv = t[q + "self_attn.v_proj.weight"]
        gate, up = t[q + "mlp.gate_proj.weight"], t[q + "mlp.up_proj.weight"]
        gu = torch.stack([gate, up], dim=1).reshape(2 * gate.shape[0], gate.shape[1])
        layers.append({
            "attn_norm": f32(t[q + "input_layernorm.weight"]),
            "wqkv": bf(torch.cat([wq, wk, wv], dim=0)),
            "wo": bf(t[q + "self_attn.o_proj.weight"]),
            "mlp_norm": f32(t[q + "post_attention_layernorm.weight"]),
            "w_gate_up": bf(gu),
            "w_down": bf(t[q + "mlp.down_proj.weight"]),
        })
    w["layers"] = layers
    return w


def load_llama(path: str, device=None, name: Optional[str] = None) -> Tuple[LlamaConfig, Dict[str, object]]:
    """(LlamaConfig, weights) from a Hugging Face Llama checkpoint directory
    (config.json + *.safetensors shards)."""
    with open(os.path.join(path, "config.json")) as fh:
        cfg = config_from_hf(json.load(fh), name or os.path.basename(os.path.normpath(path)))
    tensors = LazyShards(sorted(glob.glob(os.path.join(path, "*.safetensors"))))
    if not len(tensors):
        raise FileNotFoundError(f"no .safetensors shards under {path}")
    return cfg, pack_hf_llama(tensors, cfg, device)
