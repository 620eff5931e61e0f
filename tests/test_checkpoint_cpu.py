"""CPU: Hugging Face Llama checkpoints -> the kernels' weight layout
(checkpoint.py).

A tiny random checkpoint in HF naming / rotate-half RoPE layout is written as
real .safetensors shards + config.json, loaded, and run through the fp32
oracle forward (the same adjacent-pair RoPE the kernels use); its logits must
equal an independent forward written in HF's own convention over the original
tensors (rotate_half RoPE, separate gate/up), to fp32 rounding.
"""

import json
import math

import pytest
import torch

CFG = {"num_hidden_layers": 2, "hidden_size": 64, "num_attention_heads": 4, "num_key_value_heads": 2,
       "intermediate_size": 96, "vocab_size": 128, "rope_theta": 10000.0, "rms_norm_eps": 1e-5}


def _hf_tensors(seed=0, tied=False):
    g = torch.Generator().manual_seed(seed)
    d, H, KV, F, V = 64, 4, 2, 96, 128
    hd = d // H

    def r(*s, std=0.1):
        return (torch.randn(*s, generator=g) * std).to(torch.bfloat16)
    t = {"model.embed_tokens.weight": r(V, d, std=1.0), "model.norm.weight": (1 + r(d)).float()}
    if not tied:
        t["lm_head.weight"] = r(V, d)
    for i in range(2):
        p = f"model.layers.{i}."
        t[p + "input_layernorm.weight"] = (1 + r(d)).float()
        t[p + "post_attention_layernorm.weight"] = (1 + r(d)).float()
        t[p + "self_attn.q_proj.weight"] = r(H * hd, d)
        t[p + "self_attn.k_proj.weight"] = r(KV * hd, d)
        t[p + "self_attn.v_proj.weight"] = r(KV * hd, d)
        t[p + "self_attn.o_proj.weight"] = r(d, H * hd)
        t[p + "mlp.gate_proj.weight"] = r(F, d)
        t[p + "mlp.up_proj.weight"] = r(F, d)
        t[p + "mlp.down_proj.weight"] = r(d, F)
    return t


def _hf_forward(t, tokens, cfg):
    """Llama forward in Hugging Face's convention (rotate_half RoPE), fp32."""
    d, H, KV = cfg["hidden_size"], cfg["num_attention_heads"], cfg["num_key_value_heads"]
    hd, eps, theta = d // H, cfg["rms_norm_eps"], cfg["rope_theta"]
    f = {k: v.float() for k, v in t.items()}
    M = len(tokens)
    pos = torch.arange(M, dtype=torch.float64)
    inv = theta ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
    ang = pos[:, None] * inv[None, :]
    cos = torch.cat([ang.cos(), ang.cos()], -1).float()[:, None, :]
    sin = torch.cat([ang.sin(), ang.sin()], -1).float()[:, None, :]

    def rot(x):
        return torch.cat([-x[..., hd // 2:], x[..., :hd // 2]], -1)

    def norm(h, gw):
        return h * torch.rsqrt((h * h).mean(-1, keepdim=True) + eps) * gw

    h = f["model.embed_tokens.weight"][torch.tensor(tokens)]
    for i in range(cfg["num_hidden_layers"]):
        p = f"model.layers.{i}."
        x = norm(h, f[p + "input_layernorm.weight"])
        q = (x @ f[p + "self_attn.q_proj.weight"].T).view(M, H, hd)
        k = (x @ f[p + "self_attn.k_proj.weight"].T).view(M, KV, hd)
        v = (x @ f[p + "self_attn.v_proj.weight"].T).view(M, KV, hd)
        q, k = q * cos + rot(q) * sin, k * cos + rot(k) * sin
        k, v = k.repeat_interleave(H // KV, 1), v.repeat_interleave(H // KV, 1)
        s = torch.einsum("mhd,chd->hmc", q, k) / math.sqrt(hd)
        s = s.masked_fill(torch.triu(torch.ones(M, M, dtype=torch.bool), 1)[None], float("-inf"))
        o = torch.einsum("hmc,chd->mhd", s.softmax(-1), v).reshape(M, H * hd)
        h = h + o @ f[p + "self_attn.o_proj.weight"].T
        x = norm(h, f[p + "post_attention_layernorm.weight"])
        gt, up = x @ f[p + "mlp.gate_proj.weight"].T, x @ f[p + "mlp.up_proj.weight"].T
        h = h + (gt / (1 + torch.exp(-gt)) * up) @ f[p + "mlp.down_proj.weight"].T
    head = f.get("lm_head.weight", f["model.embed_tokens.weight"])
    return norm(h, f["model.norm.weight"]) @ head.T


@pytest.mark.parametrize("tied", [False, True])
def test_hf_checkpoint_roundtrip_matches_hf_forward(tmp_path, tied):
    from paper_2408_11850_b200 import checkpoint
    from oracle.llama import OracleLlama
    t = _hf_tensors(1, tied)
    names = sorted(t)
    checkpoint.write_safetensors(str(tmp_path / "model-00001-of-00002.safetensors"),
                                 {k: t[k] for k in names[: len(names) // 2]})
    checkpoint.write_safetensors(str(tmp_path / "model-00002-of-00002.safetensors"),
                                 {k: t[k] for k in names[len(names) // 2:]})
    (tmp_path / "config.json").write_text(json.dumps(CFG))
    cfg, w = checkpoint.load_llama(str(tmp_path))
    assert (cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.vocab) == (2, 64, 4, 2, 96, 128)
    assert w["layers"][0]["wqkv"].shape == (8 * 16, 64) and w["layers"][0]["w_gate_up"].shape == (192, 64)
    # SwiGLU interleave: rows 2j / 2j+1 are gate_j / up_j
    assert torch.equal(w["layers"][1]["w_gate_up"][0::2], t["model.layers.1.mlp.gate_proj.weight"])
    assert torch.equal(w["layers"][1]["w_gate_up"][1::2], t["model.layers.1.mlp.up_proj.weight"])
    tokens = [3, 77, 5, 120, 9, 9, 64, 1]
    ours = OracleLlama(cfg, w, bf16_points=False, max_seq=32).forward(tokens, 0)
    ref = _hf_forward(t, tokens, CFG)
    assert (ours - ref).abs().max().item() < 2e-4 * (1 + ref.abs().max().item())


def test_safetensors_reader_roundtrip(tmp_path):
    from paper_2408_11850_b200 import checkpoint
    t = {"a": torch.randn(3, 5), "b": torch.randn(7).to(torch.bfloat16), "c": torch.randn(2, 2).half()}
    p = str(tmp_path / "x.safetensors")
    checkpoint.write_safetensors(p, t)
    back = checkpoint.read_safetensors(p)
    assert set(back) == set(t)
    for k in t:
        assert back[k].dtype == t[k].dtype and torch.equal(back[k], t[k])


@pytest.mark.gpu
@pytest.mark.parametrize("gemm", ["tcgen05", "cudacore"])
def test_hf_checkpoint_runs_on_the_kernels(tmp_path, gemm):
    """A loaded HF checkpoint (head_dim 64) through the B200 forward matches the
    fp32 oracle on the same tensors within the logits tolerance of
    tests/test_llama_gpu.py."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import checkpoint, llama
    from oracle.llama import OracleLlama
    cfg_hf = dict(CFG, hidden_size=256, num_attention_heads=4, num_key_value_heads=2, intermediate_size=512,
                  vocab_size=1024)
    g = torch.Generator().manual_seed(3)
    d, F, V = 256, 512, 1024
    t = {"model.embed_tokens.weight": (torch.randn(V, d, generator=g)).to(torch.bfloat16),
         "model.norm.weight": torch.ones(d), "lm_head.weight": (torch.randn(V, d, generator=g) * 0.05).to(torch.bfloat16)}
    for i in range(2):
        p = f"model.layers.{i}."
        for n, shape in (("self_attn.q_proj", (256, d)), ("self_attn.k_proj", (128, d)), ("self_attn.v_proj", (128, d)),
                         ("self_attn.o_proj", (d, 256)), ("mlp.gate_proj", (F, d)), ("mlp.up_proj", (F, d)),
                         ("mlp.down_proj", (d, F))):
            t[p + n + ".weight"] = (torch.randn(*shape, generator=g) * 0.05).to(torch.bfloat16)
        t[p + "input_layernorm.weight"] = torch.ones(d)
        t[p + "post_attention_layernorm.weight"] = torch.ones(d)
    checkpoint.write_safetensors(str(tmp_path / "model.safetensors"), t)
    (tmp_path / "config.json").write_text(json.dumps(cfg_hf))
    cfg, w = checkpoint.load_llama(str(tmp_path), device="cuda")
    m = llama.LlamaModel(cfg, w, gemm=gemm, max_seq=64, max_tokens=32)
    toks = [1, 5, 900, 17, 4, 4, 300, 12, 1000, 2]
    got = m.forward_logits(toks).cpu()
    want = OracleLlama(cfg, w, device="cuda", bf16_points=True, max_seq=64, norm_fold=gemm == "tcgen05").forward(toks, 0).cpu()
    assert ((got - want).abs() <= 5e-2 + 1e-2 * want.abs()).all()


ROPE_CASES = [
    # DeepSeek-Coder 1.3B / 33B: linear scaling, factor 4
    (2048, 16, 100000.0, {"type": "linear", "factor": 4.0}),
    # Llama-3.1 8B / 70B: llama3 scaling
    (4096, 32, 500000.0, {"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                          "original_max_position_embeddings": 8192}),
    (8192, 64, 500000.0, {"rope_type": "llama3", "factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                          "original_max_position_embeddings": 8192}),
]


@pytest.mark.parametrize("d,H,theta,rs", ROPE_CASES)
def test_rope_scaling_matches_transformers(d, H, theta, rs):
    """config.json rope_scaling -> the kernels' RoPE tables: inverse
    frequencies equal transformers' own rope-init functions (the convention
    the checkpoints were trained with), and the oracle's independent
    restatement equals both."""
    import numpy as np
    tr = pytest.importorskip("transformers")
    from transformers.modeling_rope_utils import ROPE_INIT_FUNCTIONS
    from paper_2408_11850_b200 import checkpoint, llama
    from oracle import llama as ol
    hf = dict(CFG, hidden_size=d, num_attention_heads=H, num_key_value_heads=H, intermediate_size=4 * d,
              vocab_size=128, rope_theta=theta, rope_scaling=rs, max_position_embeddings=131072)
    cfg = checkpoint.config_from_hf(hf)
    assert cfg.rope_scaling is not None and cfg.rope_scaling[0] == rs.get("rope_type", rs.get("type"))
    kind = cfg.rope_scaling[0]
    tc = tr.LlamaConfig(hidden_size=d, num_attention_heads=H, rope_theta=theta, rope_scaling=dict(rs),
                        max_position_embeddings=131072)
    want, _ = ROPE_INIT_FUNCTIONS[kind](tc, "cpu")
    ours = llama.rope_inv_freq(d // H, theta, cfg.rope_scaling)
    assert np.allclose(ours, want.double().numpy(), rtol=1e-6, atol=0)
    orc = ol._scaled_inv_freq(theta ** (-np.arange(0, d // H, 2, dtype=np.float64) / (d // H)), cfg.rope_scaling)
    assert np.allclose(orc, ours, rtol=1e-12, atol=0)
    cos, sin = llama.rope_tables(d // H, 64, theta, cfg.rope_scaling)
    assert np.allclose(cos[37], np.cos(37 * ours).astype(np.float32))


def test_rope_scaling_unsupported_types_are_rejected():
    from paper_2408_11850_b200 import checkpoint
    for rs in ({"type": "dynamic", "factor": 2.0}, {"rope_type": "yarn", "factor": 4.0}):
        with pytest.raises(ValueError, match="rope_scaling"):
            checkpoint.config_from_hf(dict(CFG, rope_scaling=rs))
    assert checkpoint.config_from_hf(dict(CFG, rope_scaling=None)).rope_scaling is None
    assert checkpoint.config_from_hf(dict(CFG, rope_scaling={"rope_type": "default"})).rope_scaling is None


def test_bos_eos_and_vocab_from_config():
    """BOS / EOS come from config.json (Llama-3: 128000 / list of EOS ids,
    DeepSeek-Coder: 32013 / 32014); absent -> BOS 1, EOS None.  A vocab that
    is not a multiple of 4 is rejected (16-byte aligned logits rows)."""
    from paper_2408_11850_b200 import checkpoint
    c = checkpoint.config_from_hf(dict(CFG, bos_token_id=128000, eos_token_id=[128001, 128008, 128009]))
    assert (c.bos_id, c.eos_id) == (128000, 128001)
    c = checkpoint.config_from_hf(dict(CFG, bos_token_id=32013, eos_token_id=32014))
    assert (c.bos_id, c.eos_id) == (32013, 32014)
    c = checkpoint.config_from_hf(dict(CFG))
    assert (c.bos_id, c.eos_id) == (1, None)
    with pytest.raises(ValueError, match="multiple of 4"):
        checkpoint.config_from_hf(dict(CFG, vocab_size=32001))


def test_lazy_shards_read_on_demand(tmp_path):
    """load_llama packs from LazyShards: tensors are read per access, so the
    host holds one layer at a time (70B checkpoints exceed host RAM twice)."""
    from paper_2408_11850_b200 import checkpoint
    t = _hf_tensors(2)
    names = sorted(t)
    checkpoint.write_safetensors(str(tmp_path / "a.safetensors"), {k: t[k] for k in names[:5]})
    checkpoint.write_safetensors(str(tmp_path / "b.safetensors"), {k: t[k] for k in names[5:]})
    lz = checkpoint.LazyShards([str(tmp_path / "a.safetensors"), str(tmp_path / "b.safetensors")])
    assert len(lz) == len(t) and "lm_head.weight" in lz and lz.get("nope") is None
    for k in names:
        assert torch.equal(lz[k], t[k])
    assert lz[names[0]].data_ptr() != lz[names[0]].data_ptr()  # nothing cached
