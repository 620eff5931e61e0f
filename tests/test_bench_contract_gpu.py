"""GPU: bench.py keeps the driver's JSON contract (one line from rank 0 with
the required keys), on the tiny pair so it runs in seconds; and the
reference arm prints its line too."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks")


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run("--pair", "tiny", "--steps", "2", "--warmup", "3", "--new", "32", "--batch-sweep", "1,2",
             "--cpu-new", "4", "--cpu-prompt", "16")
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert "workload" in d["config"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"]
    assert d["gpu_launches"] > 0
    assert set(d["batch_sweep"]["by_batch"]) == {"1", "2"}
    assert d["run_summary"]["pearl"]["total_new_tokens"] == 2 * 32


def test_reference_arm_line():
    d = _run("--impl", "reference", "--pair", "tiny", "--steps", "1", "--warmup", "1", "--new", "8",
             "--prompt", "16", "--ref-gamma", "4")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    # the reference arm runs the GPU arm's workload: same pair, prompt and new tokens
    assert (d["config"]["pair"], d["config"]["prompt_len"], d["config"]["new_tokens"]) == ("tiny", 16, 8)


def test_bench_split_pairs_four_ranks_one_gpu():
    """N = 4 under torchrun: two split pairs (targets on ranks 0 / 2, drafts
    on 1 / 3) -- functional run with all ranks on cuda:0 over gloo
    (PEARL_BENCH_BACKEND=gloo); rank 0 prints one line whose value counts
    both pairs' tokens."""
    import socket
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, PEARL_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "4",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
                          "--gpus", "4", "--pair", "tiny", "--steps", "2", "--warmup", "1", "--new", "24",
                          "--gamma-max", "8"], capture_output=True, text=True, timeout=900, cwd=REPO, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 4 and d["config"]["global_batch"] == 2
    assert "split pairs x2" in d["config"]["parallelism"]
    assert d["value"] > 0 and d["speedup_vs_ar"] > 0
    assert d["roofline"]["frac"] > 0 and d["draft_roofline"]["us_per_launch"] > 0
