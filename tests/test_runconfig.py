"""Run configs -> engines (runconfig.py).

CPU: schema errors carry the JSON path and map to the CLI's exit codes.
GPU (every pick and verification runs in libpearl_b200, also for the
synthetic plugin models): the reference CLI's own artifacts
(tests/golden/run_cases.json, made by tests/golden/make_run_golden.py running
pearl_lab.cli ``run``) are reproduced byte for byte from the same
synthetic-family configs; a ``transformer`` config runs the device fast path,
its artifacts equal direct per-prompt decodes, and ``batch`` (lockstep
decoding) changes nothing.
"""

import json
import os

import pytest

from conftest import load_golden


def _write_case(tmp_path, case, prompts):
    doc = {k: v for k, v in case.items() if k != "no_prompts"}
    if not case.get("no_prompts"):
        p = tmp_path / "prompts.txt"
        p.write_text("\n".join(prompts) + "\n", encoding="utf-8")
        doc["prompts"] = str(p)
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(doc))
    return str(cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(5))
def test_synthetic_run_matches_reference_cli(tmp_path, ci):
    from paper_2408_11850_b200 import runconfig
    gold = load_golden("run_cases.json")
    case = gold["cases"][ci]
    cfg = _write_case(tmp_path, case["config"], gold["prompts"])
    out = tmp_path / "out"
    assert runconfig.main(["run", "--config", cfg, "--out", str(out)]) == 0
    got = {f: (out / f).read_text(encoding="utf-8") for f in sorted(os.listdir(out))}
    assert sorted(got) == sorted(case["files"])
    for name, text in case["files"].items():
        assert got[name] == text, name


def _doc(**over):
    d = {"engine": "pearl", "gamma": 4, "max_new_tokens": 8, "seed": 0,
         "model": {"transformer": {"arch": "tiny"}}}
    d.update(over)
    return d


@pytest.mark.parametrize("doc,path", [
    (_doc(bogus=1), "$"),
    (_doc(gamma=0), "$.gamma"),
    ({k: v for k, v in _doc().items() if k != "gamma"}, "$.gamma"),
    (_doc(model={"transformer": {"arch": "tiny", "dtype": "fp8"}}), "$.model.transformer.dtype"),
    (_doc(model={"transformer": {"arch": "gpt-5"}}), "$.model.transformer.arch"),
    (_doc(model={"transformer": {}}), "$.model.transformer"),
    (_doc(model={"transformer": {"arch": "tiny", "checkpoint": {"target": "a", "draft": "b"}}}),
     "$.model.transformer"),
    (_doc(model={"transformer": {"arch": "tiny", "devices": [0, 1]}}), "$.model.transformer.devices"),
    (_doc(model={"synthetic": {"alpha": 0.5}}), "$.timing"),
    (_doc(model={"synthetic": {"alpha": 1.5}}, timing={"t": 1, "c": 2}), "$.model.synthetic.alpha"),
    (_doc(model={"synthetic": {"alpha": 0.5}, "transformer": {"arch": "tiny"}}), "$.model"),
    (_doc(prompts="p.txt", synthetic_prompts={"n": 1, "length": 4, "seed": 0}), "$.synthetic_prompts"),
    (_doc(timing={"t": 0, "c": 2}), "$.timing.t"),
    (_doc(batch=4, adaptive_gamma=True), "$.adaptive_gamma"),
])
def test_config_errors_carry_json_path(doc, path):
    from paper_2408_11850_b200 import runconfig
    with pytest.raises(runconfig.ConfigError) as ei:
        runconfig.parse_run_config(doc)
    assert ei.value.path == path


def test_exit_codes(tmp_path):
    from paper_2408_11850_b200 import runconfig
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert runconfig.main(["run", "--config", str(bad), "--out", str(tmp_path / "o")]) == 2
    assert runconfig.main(["run", "--config", str(tmp_path / "missing.json"), "--out", str(tmp_path / "o")]) == 3
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"engine": "ar", "max_new_tokens": 4, "seed": 0, "prompts": str(tmp_path / "nope.txt"),
                               "model": {"synthetic": {"alpha": 0.5}}, "timing": {"t": 1, "c": 2}}))
    assert runconfig.main(["run", "--config", str(cfg), "--out", str(tmp_path / "o")]) == 3
    nodir = tmp_path / "n.json"
    nodir.write_text(json.dumps({"engine": "ar", "max_new_tokens": 4, "seed": 0,
                                 "model": {"synthetic": {"alpha": 0.5}}, "timing": {"t": 1, "c": 2}}))
    assert runconfig.main(["run", "--config", str(nodir)]) == 2
    # a decode that needs more KV positions than the kernels hold is a config error, not a traceback
    (tmp_path / "long.txt").write_text(" ".join(["5"] * 3000) + "\n")
    big = tmp_path / "big.json"
    big.write_text(json.dumps(_doc(max_new_tokens=2000, prompts=str(tmp_path / "long.txt"))))
    assert runconfig.main(["run", "--config", str(big), "--out", str(tmp_path / "o")]) == 2


@pytest.mark.gpu
def test_seed_override_and_derived_seeds(tmp_path):
    """--seed replaces the config seed; prompt i decodes with derive_seed(seed, i) (cli.py:94-96, 185-186)."""
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import runconfig
    doc = {"engine": "sd", "gamma": 3, "max_new_tokens": 20, "seed": 1, "model": {"synthetic": {"alpha": 0.7}},
           "timing": {"t": 1, "c": 4}}
    (tmp_path / "c.json").write_text(json.dumps(doc))
    assert runconfig.main(["run", "--config", str(tmp_path / "c.json"), "--out", str(tmp_path / "o"), "--seed", "9"]) == 0
    pair = pk.make_alpha_pair(0.7, 64, draft_time=1.0, target_time=4.0)
    want = pk.decode_sd(pair.draft, pair.target, [], pk.EngineConfig(gamma=3, max_new_tokens=20,
                                                                      seed=runconfig.derive_seed(9, 0)))
    assert (tmp_path / "o" / "outputs.txt").read_text().split() == [str(t) for t in want.tokens]


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["pearl", "sd", "ar"])
def test_transformer_run_on_device(tmp_path, engine):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from dataclasses import replace

    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import runconfig
    doc = {"engine": engine, "gamma": 4, "max_new_tokens": 24, "seed": 5, "greedy": False,
           "model": {"transformer": {"arch": "tiny", "gemm": "tcgen05"}},
           "synthetic_prompts": {"n": 3, "length": 9, "seed": 2}}
    cfg = runconfig.parse_run_config(doc)
    models = runconfig.build_models(replace(cfg, batch=3), max_seq=128)  # KV slots for the batch run
    draft, target, _, timing = models
    s1 = runconfig.run(cfg, str(tmp_path / "b1"), models=models)
    s3 = runconfig.run(replace(cfg, batch=3), str(tmp_path / "b3"), models=models)
    assert s1.n_prompts == 3 and s1.total_new_tokens == 3 * 24 and s1.sim_speedup > 0
    assert (s3.total_steps, s3.acceptance) == (s1.total_steps, s1.acceptance)
    out1 = (tmp_path / "b1" / "outputs.txt").read_text()
    assert out1 == (tmp_path / "b3" / "outputs.txt").read_text()
    for i in range(3):
        assert (tmp_path / "b1" / f"trace_{i:03d}.jsonl").read_text().count("\n") > 0
    prompts = runconfig.load_prompts(cfg, target.vocab_size)
    for i, line in enumerate(out1.splitlines()):
        ecfg = pk.EngineConfig(gamma=4, max_new_tokens=24, seed=runconfig.derive_seed(5, i))
        fn = {"pearl": lambda p: pk.decode_pearl(draft, target, p, ecfg),
              "sd": lambda p: pk.decode_sd(draft, target, p, ecfg),
              "ar": lambda p: pk.decode_autoregressive(target, p, ecfg)}[engine]
        assert line.split() == [str(t) for t in fn(prompts[i]).tokens]
    js = json.loads((tmp_path / "b1" / "run_summary.json").read_text())
    assert js["engine"] == engine and js["total_new_tokens"] == 72
    assert timing.c > 1.0  # measured on the GPU: the target forward costs more than the draft's


@pytest.mark.gpu
def test_transformer_checkpoint_run(tmp_path):
    """``checkpoint`` instead of ``arch``: Hugging Face safetensors for target and
    draft (checkpoint.load_llama) decoded end to end from a run config."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import checkpoint, runconfig
    d, F, V = 256, 512, 1024
    for name, seed, layers in (("target", 1, 2), ("draft", 2, 1)):
        g = torch.Generator().manual_seed(seed)

        def r(*s, std=0.05):
            return (torch.randn(*s, generator=g) * std).to(torch.bfloat16)
        t = {"model.embed_tokens.weight": r(V, d, std=1.0), "model.norm.weight": torch.ones(d),
             "lm_head.weight": r(V, d)}
        for i in range(layers):
            p = f"model.layers.{i}."
            for n, shape in (("self_attn.q_proj", (256, d)), ("self_attn.k_proj", (128, d)),
                             ("self_attn.v_proj", (128, d)), ("self_attn.o_proj", (d, 256)),
                             ("mlp.gate_proj", (F, d)), ("mlp.up_proj", (F, d)), ("mlp.down_proj", (d, F))):
                t[p + n + ".weight"] = r(*shape)
            t[p + "input_layernorm.weight"] = torch.ones(d)
            t[p + "post_attention_layernorm.weight"] = torch.ones(d)
        (tmp_path / name).mkdir()
        checkpoint.write_safetensors(str(tmp_path / name / "model.safetensors"), t)
        (tmp_path / name / "config.json").write_text(json.dumps(
            {"num_hidden_layers": layers, "hidden_size": d, "num_attention_heads": 4, "num_key_value_heads": 2,
             "intermediate_size": F, "vocab_size": V, "bos_token_id": 7, "eos_token_id": [1000, 1001],
             "rope_scaling": {"type": "linear", "factor": 4.0}}))
    (tmp_path / "p.txt").write_text("5 17 300 9\n\n900 31 2\n")  # the empty line decodes from BOS
    doc = {"engine": "pearl", "gamma": 3, "max_new_tokens": 20, "seed": 4, "prompts": str(tmp_path / "p.txt"),
           "model": {"transformer": {"checkpoint": {"target": str(tmp_path / "target"),
                                                    "draft": str(tmp_path / "draft")}}}}
    (tmp_path / "cfg.json").write_text(json.dumps(doc))
    # BOS / EOS / rope_scaling come from config.json
    draft, target, eos_id, _ = runconfig.build_models(runconfig.load_run_config(str(tmp_path / "cfg.json")),
                                                      max_seq=64)
    assert (target.bos_id, draft.bos_id, eos_id) == (7, 7, 1000)
    assert target.cfg.rope_scaling == ("linear", 4.0)
    del draft, target
    assert runconfig.main(["run", "--config", str(tmp_path / "cfg.json"), "--out", str(tmp_path / "o")]) == 0
    out = (tmp_path / "o" / "outputs.txt").read_text().splitlines()
    # 20 tokens each, or fewer ending at the checkpoint's EOS (1000)
    assert len(out) == 3 and all(len(line.split()) == 20 or line.split()[-1] == "1000" for line in out)
    assert all(0 <= int(x) < V for line in out for x in line.split())
