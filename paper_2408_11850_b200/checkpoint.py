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


def read_safetensors(path: str) -> Dict[str, torch.Tensor]:
    """All tensors of one .safetensors file as CPU torch tensors."""
    with open(path, "rb") as fh:
        (n,) = struct.unpack("<Q", fh.read(8))
        header = json.loads(fh.read(n))
        base = 8 + n
        out: Dict[str, torch.Tensor] = {}
        for name, meta in header.items():
            if name == "__metadata__":
                continue
            dt = meta["dtype"]
            if dt not in _DTYPES:
                raise ValueError(f"{path}: tensor {name} has unsupported dtype {dt}")
            tdt, size = _DTYPES[dt]
            lo, hi = meta["data_offsets"]
            fh.seek(base + lo)
            raw = bytearray(fh.read(hi - lo))
            t = torch.frombuffer(raw, dtype=tdt) if raw else torch.empty(0, dtype=tdt)
            out[name] = t.reshape(meta["shape"])
    return out


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


def config_from_hf(cfg: dict, name: str = "hf-llama") -> LlamaConfig:
    """LlamaConfig from a Hugging Face config.json (LlamaForCausalLM)."""
    H = int(cfg["num_attention_heads"])
    d = int(cfg["hidden_size"])
    hd = int(cfg.get("head_dim", d // H))
    if hd * H != d:
        raise ValueError("head_dim * num_attention_heads must equal hidden_size")
    return LlamaConfig(name, int(cfg["num_hidden_layers"]), d, H, int(cfg.get("num_key_value_heads", H)),
                       int(cfg["intermediate_size"]), int(cfg["vocab_size"]),
                       rope_theta=float(cfg.get("rope_theta", 10000.0)), norm_eps=float(cfg.get("rms_norm_eps", 1e-5)))


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
    emb = t[p + "embed_tokens.weight"]
    head = t.get("lm_head.weight", emb)
    w: Dict[str, object] = {"embed": bf(emb), "lm_head": bf(head), "final_norm": f32(t[p + "norm.weight"])}
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
    tensors: Dict[str, torch.Tensor] = {}
    for f in sorted(glob.glob(os.path.join(path, "*.safetensors"))):
        tensors.update(read_safetensors(f))
    if not tensors:
        raise FileNotFoundError(f"no .safetensors shards under {path}")
    return cfg, pack_hf_llama(tensors, cfg, device)
