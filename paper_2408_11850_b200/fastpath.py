r"""Device-resident decode loops for GPU models (the engines' fast path).

One PEARL step (engines.py:397-526) is a single CUDA graph:

    assemble  : target window [committed[-1]] + pending, draft catch-up ids
    fork ---- draft stream : gamma x (draft forward M=1 -> inverse-CDF pick)    (K2 + pick)
         \--- target stream: target forward over the window (M = k+1)         (K3/K4)
    join (event rendezvous, the _PhaseRunner of engines.py:241-262)
    K1        : fused verify of chain = pending + [x_0] (logits rows, fp64 law)
    commit    : append accepted + correction, K5 KV rollback, carry pending,
                flip PRE/POST (engines.py:431-446, 500-515)
    D2H       : a 16+gamma int summary into pinned memory

The host replays the graph for the current (k, gamma, m0) shape, waits for
the summary and builds the StepTrace -- one sync per step.  SD
(engines.py:344-394) and AR (engines.py:289-319) use the same kernels: SD as
one serial graph per step, AR as graphs of 1/2/4/8 back-to-back steps.
Uniforms come from the same split PCG64 streams as the reference, uploaded
as tables and consumed through device cursors, so a seed gives the
reference's tokens and traces.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _device, _lib
from .core import RandomStream
from .llama import LlamaModel, inv_temp

_FWD_ADVANCE = 1
_FWD_LAST = 2
U_TABLE = 4096

# pearl_seq_state field offsets (int32)
S_COMMITTED, S_NPENDING, S_MODE, S_TPOS, S_DPOS, S_VCUR, S_DCUR, S_STATUS = range(8)
# summary offsets (engine.cu SUM_*)
SUM_STATUS, SUM_ACCEPTED, SUM_CORRECTION, SUM_EXAMINED, SUM_DRAWS, SUM_BONUS, SUM_COMMITTED, SUM_MODE, \
    SUM_NPENDING, SUM_TPOS, SUM_DPOS, SUM_VCUR, SUM_DCUR, SUM_FALLBACK = range(14)
SUM_HDR = 16


class _VerifyResultC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("status", "accepted", "correction", "examined", "draws_used", "bonus", "fallback", "reserved")]


class _CommitArgs(ctypes.Structure):
    _fields_ = [("state", ctypes.c_void_p), ("seq_tokens", ctypes.c_void_p), ("max_len", ctypes.c_int32),
                ("chain", ctypes.c_void_p), ("k", ctypes.c_int32), ("gamma", ctypes.c_int32),
                ("verdict", ctypes.c_void_p), ("pending_tok", ctypes.c_void_p), ("pending_rows", ctypes.c_void_p),
                ("draft_rows", ctypes.c_void_p), ("V", ctypes.c_int32), ("sd_mode", ctypes.c_int32),
                ("out_host_view", ctypes.c_void_p)]


def _addr(t: torch.Tensor, i: int = 0) -> int:
    return int(t.data_ptr()) + i * t.element_size()


class PairRuntime:
    """Buffers and captured step graphs for one (draft, target) pair (or a target alone for AR)."""

    def __init__(self, target: LlamaModel, draft: Optional[LlamaModel], gamma_max: int):
        self.target, self.draft = target, draft
        self.dev = target.device
        V = target.cfg.vocab
        if draft is not None and draft.cfg.vocab != V:
            raise ValueError("draft and target must share a vocabulary")
        self.V = V
        self.gmax = int(gamma_max)
        self.max_len = target.max_seq
        if draft is not None:
            self.max_len = min(self.max_len, draft.max_seq)
        dev, g = self.dev, self.gmax
        i32 = dict(dtype=torch.int32, device=dev)
        self.state = torch.zeros(8, **i32)
        self.seq = torch.zeros(self.max_len + 2 * g + 4, **i32)
        self.pending_tok = torch.zeros(g + 1, **i32)
        self.pending_rows = torch.zeros(g + 1, V, dtype=torch.float32, device=dev)
        self.draft_rows = torch.zeros(g + 1, V, dtype=torch.float32, device=dev)
        self.target_rows = torch.zeros(g + 2, V, dtype=torch.float32, device=dev)
        self.target_in = torch.zeros(g + 2, **i32)
        self.chain = torch.zeros(2 * g + 2, **i32)
        self.draft_in = torch.zeros(g + 4, **i32)
        self.draft_cnt = torch.zeros(1, **i32)
        self.verdict = torch.zeros(8, **i32)
        self.summary = torch.zeros(SUM_HDR + g + 8, **i32)
        self.summary_host = torch.zeros(SUM_HDR + g + 8, dtype=torch.int32).pin_memory()
        self.u_draft = torch.zeros(U_TABLE, dtype=torch.float64, device=dev)
        self.u_verify = torch.zeros(U_TABLE, dtype=torch.float64, device=dev)
        wb = int(_lib.load().pearl_verify_work_bytes(g + 2))
        self.work_v = torch.zeros(wb, dtype=torch.uint8, device=dev)
        self.work_s = torch.zeros(wb, dtype=torch.uint8, device=dev)
        self.sample_status = torch.zeros(1, **i32)
        self.draft_row_ptrs = _device.row_ptrs([self.draft_rows[j] for j in range(g + 1)], dev)
        self.target_row_ptrs = _device.row_ptrs([self.target_rows[j] for j in range(g + 2)], dev)
        # q rows for a chain of k pending + 1 fresh: pending_rows[0..k-1], draft_rows[0]
        self.q_row_ptrs = {k: _device.row_ptrs([self.pending_rows[j] for j in range(k)] + [self.draft_rows[0]], dev)
                           for k in range(g + 1)}
        # AR
        self.ar_tok = torch.zeros(1, **i32)
        self.ar_out = torch.zeros(8, **i32)
        self.ar_out_host = torch.zeros(8, dtype=torch.int32).pin_memory()
        self.graphs: Dict[tuple, torch.cuda.CUDAGraph] = {}
        self.graph_launches: Dict[tuple, int] = {}
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        green = getattr(target, "green_partition", None)
        if green is not None:
            # each model on its own SM partition (llama.build_pair(draft_sms=...))
            self.draft_stream = torch.cuda.ExternalStream(green[0], device=dev)
            self.target_stream = torch.cuda.ExternalStream(green[1], device=dev)
        else:
            # shared SMs: stream priorities of the two concurrent models (PEARL_PRIO: draft | target |
            # none).  Equal priorities measured best with the 1-CTA/SM deep-ring GEMMs (7B/68M
            # post-verify step, gamma 16: none 4.37 ms, draft-first 4.63, target-first 4.93).
            prio = os.environ.get("PEARL_PRIO", "none")
            self.draft_stream = torch.cuda.Stream(device=dev, priority=-1 if prio == "draft" else 0)
            self.target_stream = torch.cuda.Stream(device=dev, priority=-1 if prio == "target" else 0)
        self.lib = _lib.load()
        _lib.prepare_vocab(V)

    # -- kernel launch helpers (all graph-capturable) ---------------------
    def _state_ptr(self, field: int) -> int:
        return _addr(self.state, field)

    def _pick(self, row_ptr_addr: int, out_addr: int, cursor_field: int, invt: float, greedy: bool,
              table: torch.Tensor, stream, append: Optional[int] = None) -> None:
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE
        _lib.check(self.lib.pearl_sample_rows(_lib.ROWS_LOGITS32, row_ptr_addr, 1, self.V, _device.ptr(table),
                                              int(table.numel()), self._state_ptr(cursor_field), invt, flags,
                                              out_addr, append, _device.ptr(self.sample_status),
                                              _device.ptr(self.work_s), _device.stream_ptr(stream)), "pick")

    def _draft_block(self, gamma: int, m0: int, xs_addr_fn, invt: float, greedy: bool, stream) -> None:
        d = self.draft
        pos = self._state_ptr(S_DPOS)
        for j in range(gamma):
            tok_addr = _device.ptr(self.draft_in) if j == 0 else xs_addr_fn(j - 1)
            n = m0 if j == 0 else 1
            _lib.check(self.lib.pearl_llama_forward(d.handle, tok_addr, n, pos, _FWD_ADVANCE | _FWD_LAST,
                                                    _addr(self.draft_rows, j * self.V), _device.stream_ptr(stream)),
                       "draft forward")
            self._pick(_addr(self.draft_row_ptrs, j), xs_addr_fn(j), S_DCUR, invt, greedy, self.u_draft, stream)

    def _verify(self, n: int, p_ptrs: torch.Tensor, q_ptrs: torch.Tensor, drafted_addr: int, invt: float,
                greedy: bool, bonus: bool, stream) -> None:
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE | (_lib.F_BONUS if bonus else 0)
        _lib.check(self.lib.pearl_spec_verify(_lib.ROWS_LOGITS32, _device.ptr(p_ptrs), _device.ptr(q_ptrs),
                                              drafted_addr, n, self.V, _device.ptr(self.u_verify),
                                              int(self.u_verify.numel()), self._state_ptr(S_VCUR), invt, flags,
                                              _device.ptr(self.verdict), None, _device.ptr(self.work_v),
                                              _device.stream_ptr(stream)), "spec_verify")

    def _commit(self, chain_addr: int, k: int, gamma: int, sd: bool, stream) -> None:
        a = _CommitArgs(self._state_ptr(0), _device.ptr(self.seq), self.max_len, chain_addr, k, gamma,
                        _device.ptr(self.verdict), _device.ptr(self.pending_tok), _device.ptr(self.pending_rows),
                        _device.ptr(self.draft_rows), self.V, 1 if sd else 0, _device.ptr(self.summary))
        _lib.check(self.lib.pearl_pearl_commit(ctypes.byref(a), _device.stream_ptr(stream)), "commit")

    def _assemble(self, stream) -> None:
        _lib.check(self.lib.pearl_step_assemble(self._state_ptr(0), _device.ptr(self.seq),
                                                _device.ptr(self.pending_tok), _device.ptr(self.target_in),
                                                _device.ptr(self.draft_in), _device.ptr(self.draft_cnt),
                                                _device.stream_ptr(stream)), "assemble")

    # -- step bodies ----------------------------------------------------------
    def _pearl_body(self, k: int, gamma: int, m0: int, invt: float, greedy: bool, concurrent: bool) -> None:
        s0 = torch.cuda.current_stream()
        self._assemble(s0)
        xs_addr = lambda j: _addr(self.chain, k + j)  # noqa: E731
        ptr_p = self.target_row_ptrs
        ptr_q = self.q_row_ptrs[k]
        tgt = self.target
        if concurrent:
            ds, ts = self.draft_stream, self.target_stream
            ds.wait_stream(s0)
            ts.wait_stream(s0)
        else:
            ds = ts = s0
        with torch.cuda.stream(ds):
            self._draft_block(gamma, m0, xs_addr, invt, greedy, ds)
        with torch.cuda.stream(ts):
            _lib.check(self.lib.pearl_llama_forward(tgt.handle, _device.ptr(self.target_in), k + 1,
                                                    self._state_ptr(S_TPOS), 0, _device.ptr(self.target_rows),
                                                    _device.stream_ptr(ts)), "target forward")
        if concurrent:
            s0.wait_stream(ds)
            s0.wait_stream(ts)
        # the chain's first k ids are the pending block: copy it in front of xs
        if k > 0:
            self.chain[:k].copy_(self.pending_tok[:k])
        self._verify(k + 1, ptr_p, ptr_q, _device.ptr(self.chain), invt, greedy, False, s0)
        self._commit(_device.ptr(self.chain), k, gamma, False, s0)
        self.summary_host.copy_(self.summary, non_blocking=True)

    def _sd_body(self, gamma: int, m0: int, invt: float, greedy: bool) -> None:
        s0 = torch.cuda.current_stream()
        self._assemble(s0)
        chain = lambda j: _addr(self.target_in, 1 + j)  # noqa: E731  (xs live right after committed[-1])
        self._draft_block(gamma, m0, chain, invt, greedy, s0)
        _lib.check(self.lib.pearl_llama_forward(self.target.handle, _device.ptr(self.target_in), gamma + 1,
                                                self._state_ptr(S_TPOS), 0, _device.ptr(self.target_rows),
                                                _device.stream_ptr(s0)), "target forward")
        q_ptrs = self.draft_row_ptrs
        self._verify(gamma, self.target_row_ptrs, q_ptrs, chain(0), invt, greedy, True, s0)
        self._commit(chain(0), 0, gamma, True, s0)
        self.summary_host.copy_(self.summary, non_blocking=True)

    def _ar_body(self, steps: int, invt: float, greedy: bool) -> None:
        s0 = torch.cuda.current_stream()
        for i in range(steps):
            _lib.check(self.lib.pearl_llama_forward(self.target.handle, _device.ptr(self.ar_tok), 1,
                                                    self._state_ptr(S_TPOS), _FWD_ADVANCE | _FWD_LAST,
                                                    _device.ptr(self.target_rows), _device.stream_ptr(s0)),
                       "target forward")
            self._pick(_addr(self.target_row_ptrs, 0), _addr(self.ar_out, i), S_VCUR, invt, greedy, self.u_verify,
                       s0, append=_device.ptr(self.ar_tok))
        self.ar_out_host.copy_(self.ar_out, non_blocking=True)

    def graph(self, key: tuple, body) -> torch.cuda.CUDAGraph:
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            c0 = int(self.lib.pearl_launch_count())
            with torch.cuda.graph(g):
                body()
            self.graph_launches[key] = int(self.lib.pearl_launch_count()) - c0
            self.graphs[key] = g
        return g

    def replay(self, key: tuple, body, stats: dict) -> float:
        """Replay the step graph for ``key``, timing it on the device (returns seconds)."""
        g = self.graph(key, body)
        self.ev[0].record()
        g.replay()
        self.ev[1].record()
        self.ev[1].synchronize()
        t = self.ev[0].elapsed_time(self.ev[1]) / 1e3
        stats["device_s"] += t
        stats["launches"] += self.graph_launches[key]
        stats["replays"] += 1
        return t

    # -- decode-level helpers ---------------------------------------------------
    def reset(self, seq0: List[int], stats: Optional[dict] = None) -> None:
        C = len(seq0)
        c0 = int(self.lib.pearl_launch_count())
        self.ev[2].record()
        if C + 2 > self.max_len:
            raise ValueError("prompt does not fit the KV cache")
        self.seq[:C].copy_(torch.tensor(seq0, dtype=torch.int32))
        st = torch.tensor([C, 0, 0, 0, 0, 0, 0, 0], dtype=torch.int32)
        self.state.copy_(st)
        # prefill both caches with all but the last committed token; the two
        # models' prefills are independent (own caches, own position fields)
        # and run concurrently on their step streams
        if C > 1:
            s0 = torch.cuda.current_stream()
            ts = self.target_stream
            ts.wait_stream(s0)
            with torch.cuda.stream(ts):
                self.target.forward(self.seq[:C - 1], C - 1, self.state[S_TPOS:S_TPOS + 1], _FWD_ADVANCE, None, ts)
            if self.draft is not None:
                ds = self.draft_stream
                ds.wait_stream(s0)
                with torch.cuda.stream(ds):
                    self.draft.forward(self.seq[:C - 1], C - 1, self.state[S_DPOS:S_DPOS + 1], _FWD_ADVANCE, None, ds)
                s0.wait_stream(ds)
            s0.wait_stream(ts)
        self.ev[3].record()
        self.ev[3].synchronize()
        if stats is not None:
            t = self.ev[2].elapsed_time(self.ev[3]) / 1e3
            stats["device_s"] += t
            stats["prefill_s"] += t
            stats["launches"] += int(self.lib.pearl_launch_count()) - c0
        self.target.reset_adapter()
        if self.draft is not None:
            self.draft.reset_adapter()

    def load_uniforms(self, table: torch.Tensor, rng: RandomStream) -> None:
        table.copy_(torch.from_numpy(np.array(rng.peek(U_TABLE))))


class _Tables:
    """Host mirror of a device uniform table + its stream."""

    def __init__(self, rt: PairRuntime, table: torch.Tensor, rng: Optional[RandomStream], field: int):
        self.rt, self.table, self.rng, self.field = rt, table, rng, field
        self.host_cursor = 0
        if rng is not None:
            rt.load_uniforms(table, rng)

    def advance(self, used_total_device: int, margin: int) -> None:
        """Refill when the device cursor gets within ``margin`` of the end."""
        self.host_cursor = used_total_device
        if self.rng is not None and used_total_device > U_TABLE - margin:
            self.rng.consume(used_total_device)
            self.rt.load_uniforms(self.table, self.rng)
            self.rt.state[self.field] = 0
            self.host_cursor = 0


def _runtime(target: LlamaModel, draft: Optional[LlamaModel], gamma_max: int) -> PairRuntime:
    cache = target.__dict__.setdefault("_pearl_runtimes", {})
    key = (id(draft), gamma_max)
    rt = cache.get(key)
    if rt is None:
        rt = PairRuntime(target, draft, gamma_max)
        cache[key] = rt
    return rt


def _new_stats(**kw) -> dict:
    d = {"device_s": 0.0, "prefill_s": 0.0, "launches": 0, "replays": 0, "fallbacks": 0}
    d.update(kw)
    return d


def _seq0(model: LlamaModel, prefix: Sequence[int]) -> List[int]:
    return [model.bos_id] + [int(t) for t in prefix]


def pearl_tokens_per_step(alpha: float, gamma: int) -> float:
    """Stationary mean tokens finalised per PEARL step under the reference's
    semantics (pre-verify finalises exactly 1, engines.py:453; post-verify
    finalises the accepted chain + correction or gamma, engines.py:500-515):
    E = (1 - a^g) / ((1 - a)(1 - a^g + a)) -- the two-state Markov chain over
    PRE/POST modes.  alpha -> 1 gives gamma."""
    a = min(max(alpha, 1e-6), 1.0 - 1e-9)
    ag = a ** gamma
    return (1.0 - ag) / ((1.0 - a) * (1.0 - ag + a))


@dataclass
class PlannerCalibration:
    """Frozen step-time model of one (draft, target) pair on one device.

    ``step_s[(pre_verify, gamma)]`` = device seconds of that PEARL step graph
    (draft catch-up m0 = 1), measured once by :func:`calibrate_planner`;
    ``alpha0`` = the pair's acceptance, the prior every decode starts from.
    With a calibration installed (:func:`set_planner_calibration`) the
    adaptive planner prices draft lengths from this table only -- no timing
    measured during a decode feeds back -- so a decode's gamma schedule is a
    function of its tokens alone and identical on every box that loads the
    same table."""

    step_s: Dict[Tuple[bool, int], float]
    alpha0: float = 0.75
    source: str = "live"

    def to_json(self) -> dict:
        return {"step_ms": {f"{'pre' if p else 'post'}:{g}": round(v * 1e3, 5) for (p, g), v in
                            sorted(self.step_s.items())},
                "alpha0": round(self.alpha0, 4), "source": self.source}

    @classmethod
    def from_json(cls, d: dict, source: str = "file") -> "PlannerCalibration":
        st = {}
        for k, v in d["step_ms"].items():
            mode, g = k.split(":")
            st[(mode == "pre", int(g))] = float(v) / 1e3
        return cls(st, float(d.get("alpha0", 0.75)), source)


def _frozen_key(draft) -> str:
    return "_pearl_frozen_" + str(id(draft))


def set_planner_calibration(draft, target, cal: Optional[PlannerCalibration]) -> None:
    """Install (or, with None, remove) a frozen planner calibration for a pair."""
    if cal is None:
        target.__dict__.pop(_frozen_key(draft), None)
    else:
        target.__dict__[_frozen_key(draft)] = cal


def calibrate_planner(draft, target, prefix: Sequence[int], gamma_max: int, temperature: float = 1.0,
                      greedy: bool = False, new_tokens: int = 96, seed: int = 12345,
                      concurrent: bool = True) -> PlannerCalibration:
    """Measure the step-time table: one fixed-gamma decode per grid gamma
    (both step kinds occur), median device time per (kind, gamma)."""
    from .engines import EngineConfig, empirical_acceptance
    prev = target.__dict__.pop(_frozen_key(draft), None)
    times: Dict[Tuple[bool, int], List[float]] = {}
    steps_all = []
    try:
        for g in [g for g in _GammaPlanner.GRID if g <= gamma_max]:
            cfg = EngineConfig(gamma=g, max_new_tokens=new_tokens, seed=seed, greedy=greedy,
                               temperature=temperature, gamma_max=max(gamma_max, g))
            for rep in range(2):  # the first decode captures the graphs
                res = decode_pearl(draft, target, prefix, cfg, concurrent=concurrent)
            for pre, gg, m0, t in res.stats["step_log"]:
                if m0 == 1:
                    times.setdefault((pre, gg), []).append(t)
            steps_all += list(res.steps)
    finally:
        if prev is not None:
            target.__dict__[_frozen_key(draft)] = prev
    step_s = {k: float(np.median(v)) for k, v in times.items()}
    # a kind never reached at some gamma (e.g. post-verify at alpha ~ 0): the
    # other kind's time, the closest proxy
    for g in [g for g in _GammaPlanner.GRID if g <= gamma_max]:
        for pre in (True, False):
            if (pre, g) not in step_s and (not pre, g) in step_s:
                step_s[(pre, g)] = step_s[(not pre, g)]
    alpha = empirical_acceptance(steps_all)
    return PlannerCalibration(step_s, float(alpha) if alpha is not None else 0.75, "live")


class _GammaPlanner:
    """Adaptive draft length (paper §3.4): gamma maximising expected PEARL
    tokens per unit of device time,

        rate(g) = E(g, alpha_hat) / (pi_pre(g) T_pre(g) + pi_post(g) T_post(g)),

    with E the stationary tokens per step (pearl_tokens_per_step), pi the
    stationary PRE / POST step shares (pi_post / pi_pre = a / (1 - a^g)) and
    alpha_hat a running Laplace estimate of this decode's acceptance.  Step
    times T are the MEASURED device times of that (mode, g) step graph when
    it has run before (EMA, kept per model pair across decodes), else the
    contention-free model max(t_target(M), g * t_draft) from one calibration
    of each model.  On a shared GPU the draft's kernels compete with the
    target's for SMs and HBM, which the model does not see; the measurements
    do (7B/68M: the model prices gamma 32 at 4.6 ms, it runs in 7.4 ms)."""

    GRID = (1, 2, 3, 4, 6, 8, 12, 16, 20, 24, 32, 48, 64)

    def __init__(self, target: LlamaModel, draft: LlamaModel, gamma_max: int, gamma0: int):
        frozen = target.__dict__.get(_frozen_key(draft))
        self.frozen = frozen is not None
        if self.frozen:
            # frozen table: no calibration forwards, no feedback from decode timings
            self.meas = dict(frozen.step_s)
            self.t_d, self.t_t = 0.0, {1: 1.0}
            self.gmax = gamma_max
            self.acc, self.exam = 8.0 * frozen.alpha0, 8.0
            self.gamma = gamma0
            self.started = False
            return
        key = "_pearl_calib_" + str(id(draft))
        cal = target.__dict__.get(key)
        if cal is None:
            green = getattr(target, "green_partition", None)
            sd = torch.cuda.ExternalStream(green[0]) if green else torch.cuda.current_stream()
            st = torch.cuda.ExternalStream(green[1]) if green else torch.cuda.current_stream()
            with torch.cuda.stream(sd):  # each model timed where PEARL runs it
                t_d = draft.measure_forward_time(1) + 6e-6  # + the pick kernel
            ms = [1, 8, 16, 32]
            with torch.cuda.stream(st):
                t_t = {m: target.measure_forward_time(m) for m in ms}
            cal = (t_d, t_t)
            target.__dict__[key] = cal
        self.t_d, self.t_t = cal
        self.meas = target.__dict__.setdefault("_pearl_steptimes_" + str(id(draft)), {})
        self.gmax = gamma_max
        # prior: 8 pseudo-observations at the pair's acceptance so far (0.75
        # before any decode), so a decode does not re-learn alpha from scratch
        self.pair = target.__dict__.setdefault("_pearl_alpha_" + str(id(draft)), [3.0, 4.0])
        a0 = self.pair[0] / self.pair[1]
        self.acc, self.exam = 8.0 * a0, 8.0
        self.gamma = gamma0
        self.started = False

    def _t_target(self, m: int) -> float:
        ks = sorted(self.t_t)
        if m <= ks[0]:
            return self.t_t[ks[0]]
        for lo, hi in zip(ks, ks[1:]):
            if m <= hi:
                w = (m - lo) / (hi - lo)
                return (1 - w) * self.t_t[lo] + w * self.t_t[hi]
        return self.t_t[ks[-1]] * m / ks[-1]

    def observe(self, accepted: int, rejected: int) -> None:
        self.acc += accepted
        self.exam += accepted + rejected
        if hasattr(self, "pair") and not self.frozen:
            self.pair[0] += accepted
            self.pair[1] += accepted + rejected

    def observe_time(self, pre: bool, g: int, seconds: float) -> None:
        """Measured device time of one step graph (co-resident path only: the
        split pair's two ranks must plan identically, so they use the model)."""
        if self.frozen:
            return
        k = (bool(pre), int(g))
        old = self.meas.get(k)
        self.meas[k] = seconds if old is None else 0.75 * old + 0.25 * seconds

    def _model_time(self, pre: bool, g: int) -> float:
        return max(self._t_target(1 if pre else g), g * self.t_d)

    def step_time(self, pre: bool, g: int) -> float:
        """Measured time of the (mode, g) step graph, else the model scaled by
        the mean measured/model ratio of the steps seen so far (so unexplored
        draft lengths are priced with the contention already observed)."""
        m = self.meas.get((bool(pre), int(g)))
        if m is not None:
            return m
        if self.frozen:  # outside the table: linear in gamma from its largest entry
            ks = [q for (p, q) in self.meas if p == bool(pre)] or [q for (_, q) in self.meas]
            g0 = max(ks)
            return self.meas.get((bool(pre), g0), self.meas.get((not pre, g0))) * g / g0
        model = self._model_time(pre, g)
        if self.meas:
            logs = [math.log(v / self._model_time(p, q)) for (p, q), v in self.meas.items()]
            model *= math.exp(sum(logs) / len(logs))
        return model

    def rate(self, alpha: float, g: int) -> float:
        a = min(max(alpha, 1e-6), 1.0 - 1e-9)
        post_per_pre = a / (1.0 - a ** g)
        t = (self.step_time(True, g) + post_per_pre * self.step_time(False, g)) / (1.0 + post_per_pre)
        return pearl_tokens_per_step(alpha, g) / t

    def candidates(self) -> List[int]:
        return [g for g in self.GRID if g <= self.gmax]

    def neighbors(self, g: int) -> List[int]:
        """Draft lengths reachable from g in one decision (itself and the grid neighbours)."""
        c = self.candidates()
        if g not in c:
            return c
        i = c.index(g)
        return c[max(0, i - 1):i + 2]

    def next_gamma(self) -> int:
        """First call: the best grid value; afterwards at most one grid step
        per decision (hysteresis), which also bounds the set of step graphs a
        decode can need (precaptured by decode_pearl)."""
        alpha = self.acc / self.exam
        best, best_rate = 1, -1.0
        cands = self.candidates() if not self.started else self.neighbors(self.gamma)
        for g in cands:
            rate = self.rate(alpha, g)
            if rate > best_rate:
                best, best_rate = g, rate
        self.gamma = best
        self.started = True
        return best


def choose_gamma(cfg, target: LlamaModel, draft: LlamaModel) -> int:
    """Initial draft length: cfg.gamma, or the planner's choice under adaptive_gamma."""
    if not cfg.adaptive_gamma:
        return cfg.gamma
    return _GammaPlanner(target, draft, cfg.gamma_max, cfg.gamma).next_gamma()


# -- engines ---------------------------------------------------------------


def decode_pearl(draft: LlamaModel, target: LlamaModel, prefix: Sequence[int], cfg, concurrent: bool = True):
    from .engines import DecodeResult, StepTrace, finalize_step
    planner = _GammaPlanner(target, draft, cfg.gamma_max, cfg.gamma) if cfg.adaptive_gamma else None
    gmax = max(cfg.gamma_max, cfg.gamma)
    t_d1 = draft.latency.forward_time  # (measured before the caches are filled)
    t_t = target.latency.forward_time
    rt = _runtime(target, draft, gmax)
    seq0 = _seq0(target, prefix)
    n0 = len(seq0)
    invt = inv_temp(cfg.temperature)
    gamma = planner.next_gamma() if planner else cfg.gamma
    stats = _new_stats(gamma=gamma, gammas=[], step_log=[])
    rt.reset(seq0, stats)
    root = RandomStream(cfg.seed)
    tab_d = _Tables(rt, rt.u_draft, None if cfg.greedy else root.split(0), S_DCUR)
    tab_v = _Tables(rt, rt.u_verify, None if cfg.greedy else root.split(1), S_VCUR)
    _precapture_pearl(rt, planner, gamma, invt, bool(cfg.greedy), bool(concurrent))
    committed: List[int] = list(seq0)
    pending: List[int] = []
    dpos = n0 - 1
    steps: List = []
    produced = 0
    while produced < cfg.max_new_tokens:
        if len(committed) + len(pending) + gamma + 2 >= rt.max_len:
            raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        k = len(pending)
        m0 = len(committed) + k - dpos
        stats["gammas"].append(gamma)
        key = ("pearl", k, gamma, m0, bool(cfg.greedy), invt, bool(concurrent))
        t_step = rt.replay(key, lambda: rt._pearl_body(k, gamma, m0, invt, cfg.greedy, concurrent), stats)
        stats["step_log"].append((k == 0, gamma, m0, t_step))
        if planner is not None and m0 == 1:
            planner.observe_time(k == 0, gamma, t_step)
        s = rt.summary_host.numpy()
        status = int(s[SUM_STATUS])
        _lib.check(status, "decode_pearl step")
        n_acc, corr = int(s[SUM_ACCEPTED]), int(s[SUM_CORRECTION])
        xs = [int(t) for t in s[SUM_HDR:SUM_HDR + gamma]]
        stats["fallbacks"] += int(s[SUM_FALLBACK])
        chain = pending + [xs[0]]
        kind = "pre_verify" if k == 0 and not steps_mode_post(steps) else "post_verify"
        if corr < 0:
            committed += chain
            pending = xs[1:]
            acc, cval, delta = k + 1, None, k + 1
        else:
            committed += chain[:n_acc] + [corr]
            pending = []
            acc, cval, delta = n_acc, corr, n_acc + 1
        dpos = int(s[SUM_DPOS])
        assert int(s[SUM_COMMITTED]) == len(committed)
        if kind == "pre_verify":
            acc = 1 if corr < 0 else 0
        trace = StepTrace(len(steps), kind, tuple(xs), acc, cval, delta, gamma * t_d1, t_t)
        if planner is not None:
            planner.observe(acc, 0 if cval is None else 1)
            gamma = planner.next_gamma()
        tab_v.advance(int(s[SUM_VCUR]), 2 * gmax + 8)
        tab_d.advance(int(s[SUM_DCUR]), 2 * gmax + 8)
        stop = finalize_step(tuple(committed), n0, produced, cfg)
        if stop is not None:
            steps.append(replace(trace, finalized_delta=stop - produced))
            return DecodeResult(tuple(committed[n0:n0 + stop]), tuple(steps), stats=stats)
        steps.append(trace)
        produced = len(committed) - n0
    return DecodeResult(tuple(committed[n0:]), tuple(steps), stats=stats)


def _precapture_pearl(rt: PairRuntime, planner, gamma: int, invt: float, greedy: bool, concurrent: bool) -> None:
    """Capture every step graph this decode can reach before it starts: keys
    (pending k, gamma, draft catch-up m0 = 1) with k = 0 (pre-verify) or
    k = gamma' - 1 for each gamma' one planner decision away (post-verify).
    Graph capture (~tens of ms each) then never lands inside a decode; rarer
    keys (m0 > 1) are still captured on first use."""
    gammas = planner.candidates() if planner is not None else [gamma]
    for g in gammas:
        prevs = planner.neighbors(g) if planner is not None else [g]
        for k in sorted({0} | {gp - 1 for gp in prevs if gp > 1}):
            key = ("pearl", k, g, 1, greedy, invt, concurrent)
            rt.graph(key, lambda k=k, g=g: rt._pearl_body(k, g, 1, invt, greedy, concurrent))


def steps_mode_post(steps) -> bool:
    """Mode the engine is in before the next step: POST iff the last step fully accepted."""
    return bool(steps) and steps[-1].correction is None


def decode_sd(draft: LlamaModel, target: LlamaModel, prefix: Sequence[int], cfg):
    from .engines import DecodeResult, StepTrace
    gamma = cfg.gamma
    t_d = gamma * draft.latency.forward_time
    t_t = target.latency.forward_time
    rt = _runtime(target, draft, max(cfg.gamma_max, gamma))
    seq0 = _seq0(target, prefix)
    n0 = len(seq0)
    stats = _new_stats(gamma=gamma)
    rt.reset(seq0, stats)
    root = RandomStream(cfg.seed)
    tab_d = _Tables(rt, rt.u_draft, None if cfg.greedy else root.split(0), S_DCUR)
    tab_v = _Tables(rt, rt.u_verify, None if cfg.greedy else root.split(1), S_VCUR)
    invt = inv_temp(cfg.temperature)
    seq: List[int] = list(seq0)
    dpos = n0 - 1
    steps: List = []
    done = False
    while not done and len(seq) - n0 < cfg.max_new_tokens:
        if len(seq) + gamma + 4 >= rt.max_len:
            raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        m0 = len(seq) - dpos
        key = ("sd", gamma, m0, bool(cfg.greedy), invt)
        rt.replay(key, lambda: rt._sd_body(gamma, m0, invt, cfg.greedy), stats)
        s = rt.summary_host.numpy()
        _lib.check(int(s[SUM_STATUS]), "decode_sd step")
        n_acc, corr, bonus = int(s[SUM_ACCEPTED]), int(s[SUM_CORRECTION]), int(s[SUM_BONUS])
        xs = [int(t) for t in s[SUM_HDR:SUM_HDR + gamma]]
        block = xs[:n_acc] + [bonus if corr < 0 else corr]
        appended = 0
        for tok in block:
            seq.append(tok)
            appended += 1
            if (cfg.eos_id is not None and tok == cfg.eos_id) or len(seq) - n0 >= cfg.max_new_tokens:
                done = True
                break
        dpos = int(s[SUM_DPOS])
        steps.append(StepTrace(len(steps), "sd", tuple(xs), min(n_acc, appended), None if corr < 0 else corr,
                               appended, t_d, t_t))
        tab_v.advance(int(s[SUM_VCUR]), 2 * gamma + 8)
        tab_d.advance(int(s[SUM_DCUR]), 2 * gamma + 8)
        stats["fallbacks"] += int(s[SUM_FALLBACK])
    return DecodeResult(tuple(seq[n0:]), tuple(steps), stats=stats)


def decode_autoregressive(target: LlamaModel, prefix: Sequence[int], cfg):
    from .engines import DecodeResult, StepTrace
    t_t = target.latency.forward_time
    rt = _runtime(target, None, max(cfg.gamma_max, cfg.gamma))
    seq0 = _seq0(target, prefix)
    n0 = len(seq0)
    stats = _new_stats()
    rt.reset(seq0, stats)
    rng = None if cfg.greedy else RandomStream(cfg.seed)
    tab = _Tables(rt, rt.u_verify, rng, S_VCUR)
    rt.ar_tok.fill_(seq0[-1])
    invt = inv_temp(cfg.temperature)
    out: List[int] = []
    steps: List = []
    while len(out) < cfg.max_new_tokens:
        remaining = cfg.max_new_tokens - len(out)
        G = 8 if remaining >= 8 else (4 if remaining >= 4 else (2 if remaining >= 2 else 1))
        if n0 + len(out) + G + 1 >= rt.max_len:
            raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        if rng is not None and int(rt.state[S_VCUR].item()) + G > U_TABLE - 8:
            tab.advance(int(rt.state[S_VCUR].item()), U_TABLE)
        key = ("ar", G, bool(cfg.greedy), invt)
        rt.replay(key, lambda: rt._ar_body(G, invt, cfg.greedy), stats)
        toks = [int(t) for t in rt.ar_out_host.numpy()[:G]]
        for tok in toks:
            out.append(tok)
            steps.append(StepTrace(len(steps), "ar", (), 0, None, 1, 0.0, t_t))
            if cfg.eos_id is not None and tok == cfg.eos_id:
                return DecodeResult(tuple(out), tuple(steps), stats=stats)
    return DecodeResult(tuple(out), tuple(steps), stats=stats)
