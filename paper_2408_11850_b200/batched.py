r"""Batched lockstep decoding of B independent prompts.

The reference decodes one prompt per engine call; its CLI runs a prompt list
as independent decodes, each with its own derived seed (cli.py:94-96,
181-208), so B > 1 must equal B independent decodes.  Here the B sequences
advance in lockstep and share every model pass:

* every target forward is ONE slot-mode pass over the concatenated windows of
  all active sequences (``pearl_llama_forward_slots``: token i at position
  tok_pos[i] of KV slot tok_slot[i]) -- the weights stream once per step for
  the whole batch, which is where batching pays on an HBM-bound decode;
* every draft iteration is one slot-mode pass over one token per sequence
  (plus the catch-up tokens after a rejection), followed by one
  ``pearl_sample_rows_multi`` launch that picks every sequence's next draft
  from its own uniform stream;
* verification is ONE K1 launch for all sequences
  (``pearl_spec_verify_multi``: each chain its own length, rows, uniform
  stream, cursor and verdict; the last draft id read on the device), then the
  host applies each sequence's PRE / POST transition.

Each sequence keeps exactly the state machine of the single-sequence engines
(engines.py:397-526 for PEARL, :344-394 SD, :289-319 AR), its own split
RandomStreams and its own KV slot.  Because every kernel computes a token's
values with an order that does not depend on which other tokens share the
launch (batch invariance), a batched decode returns, token for
token and step for step, what ``decode_pearl`` / ``decode_sd`` /
``decode_autoregressive`` return for each prompt alone
(tests/test_batched_gpu.py).

Draft length is fixed (cfg.gamma) in batched mode.
"""

from __future__ import annotations

from dataclasses import replace
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _device, _lib
from .core import RandomStream
from .llama import LlamaModel, inv_temp

U_TABLE = 4096


def derive_seed(seed: int, index: int) -> int:
    """Per-prompt seed of the reference CLI (cli.py:94-96)."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(index,))
    return int(ss.generate_state(1, np.uint64)[0])


class _Seq:
    """Host mirror of one sequence's DecodeState (engines.py:80-99)."""

    def __init__(self, slot: int, seq0: List[int], cfg):
        self.slot = slot
        self.cfg = cfg
        self.n0 = len(seq0)
        self.committed: List[int] = list(seq0)
        self.pending: List[int] = []
        self.pending_q: List[int] = []  # device addresses of the pending drafts' q rows
        self.dpos = self.n0 - 1          # draft KV length
        self.steps: List = []
        self.done = False
        self.tokens: Optional[tuple] = None
        self.dcur = 0                    # host mirrors of the device uniform cursors
        self.vcur = 0


class BatchRuntime:
    """Device buffers of one (target, draft) pair decoding up to B sequences."""

    def __init__(self, target: LlamaModel, draft: Optional[LlamaModel], B: int, gamma_max: int):
        if target.n_slots < B or (draft is not None and draft.n_slots < B):
            raise ValueError(f"models need n_slots >= {B} (llama.build_pair(..., n_slots=B))")
        if draft is not None and draft.cfg.vocab != target.cfg.vocab:
            raise ValueError("draft and target must share a vocabulary")
        self.target, self.draft, self.B, self.g = target, draft, int(B), int(gamma_max)
        self.V = V = target.cfg.vocab
        self.dev = dev = target.device
        self.max_len = min(target.max_seq, draft.max_seq) if draft is not None else target.max_seq
        g, i32 = self.g, dict(dtype=torch.int32, device=dev)
        self.lib = _lib.load()
        _lib.prepare_vocab(V)
        # per-sequence uniform tables and cursors ([0] draft stream, [1] verify stream)
        self.tables = torch.zeros(2, B, U_TABLE, dtype=torch.float64, device=dev)
        self.cursors = torch.zeros(2, B, **i32)
        # draft logits: iteration 0 (catch-up rows) in `stage`; iteration j >= 1
        # in qbuf[parity, j, rank] (kept one extra step as the pending q rows)
        self.stage = torch.zeros(B * (g + 2), V, dtype=torch.float32, device=dev)
        self.qbuf = torch.zeros(2, g + 1, B, V, dtype=torch.float32, device=dev)
        self.trows = torch.zeros(B * (g + 2), V, dtype=torch.float32, device=dev)
        self.xs = torch.zeros(g + 1, B, **i32)
        self.verdict = torch.zeros(B, 8, **i32)
        self.status = torch.zeros(1, **i32)
        wb = int(self.lib.pearl_verify_work_bytes(g + 2))
        self.work = torch.zeros(B, wb, dtype=torch.uint8, device=dev)
        # per-step index buffers, filled from one pinned host staging array
        # (sized for the largest upload: a prefill of every slot's full context)
        self.ibuf = torch.zeros(2 * B * self.max_len + 16 * B * (g + 2) * (g + 2) + 4096, dtype=torch.int64, device=dev)
        self.ibuf_host = torch.zeros_like(self.ibuf, device="cpu").pin_memory()
        self.out_host = torch.zeros(B * 8 + (g + 1) * B + 2 * B + 1, dtype=torch.int32).pin_memory()
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        self.draft_stream = torch.cuda.Stream(device=dev)
        self.target_stream = torch.cuda.Stream(device=dev)
        self.graphs = {}
        self.tcap = B * (g + 2)  # target window tokens per step (max)

    # -- helpers ----------------------------------------------------------------
    def load_table(self, s: int, i: int, rng: RandomStream) -> None:
        self.tables[s, i].copy_(torch.from_numpy(np.array(rng.peek(U_TABLE))))

    def begin_step(self) -> None:
        """Uploads of one step take consecutive regions of the staging slabs
        (the previous step's copies completed at its read-back sync)."""
        self._off = 0

    def upload(self, chunks: List[np.ndarray], caps: Optional[List[int]] = None) -> List[torch.Tensor]:
        """Copy int arrays to the device in one transfer on the current stream;
        returns device views (int32 arrays become int32 views of the int64 slab).
        With `caps`, chunk i occupies cap[i] elements whatever its length, so a
        fixed sequence of capped uploads at the start of a step lands at fixed
        device addresses (the inputs of the captured step graphs)."""
        host = self.ibuf_host.numpy()
        views, off = [], getattr(self, "_off", 0)
        start = off
        for ci, a in enumerate(chunks):
            n = len(a)
            cap = max(n, caps[ci]) if caps is not None else n
            if caps is not None and n > caps[ci]:
                raise ValueError("batched upload exceeds its capped region")
            if a.dtype == np.int64:
                host[off:off + n] = a
                views.append(("i64", off, n))
                off += cap
            else:
                m = (cap + 1) // 2
                host[off:off + (n + 1) // 2].view(np.int32)[:n] = a.astype(np.int32)
                views.append(("i32", off, n))
                off += m
        if off > len(host):
            raise ValueError("batched index buffer overflow")
        self.ibuf[start:off].copy_(self.ibuf_host[start:off], non_blocking=True)
        self._off = off
        out = []
        for kind, o, n in views:
            if kind == "i64":
                out.append(self.ibuf[o:o + n])
            else:
                out.append(self.ibuf[o:o + (n + 1) // 2].view(torch.int32)[:n])
        return out

    def stream_ptrs(self, sel: int, act: List["_Seq"]) -> np.ndarray:
        """Per-rank (table, cursor) addresses of the active sequences' `sel` stream."""
        t = [int(self.tables[sel, s.slot].data_ptr()) for s in act]
        c = [_addr(self.cursors[sel], s.slot) for s in act]
        return np.array(t + c, np.int64)

    def pick(self, rows_ptrs: torch.Tensor, n: int, out_addr: int, sptrs: torch.Tensor, invt: float, greedy: bool,
             stream) -> None:
        """One pick per active sequence; row r uses rank r's own stream (sptrs = stream_ptrs(...) on device)."""
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE
        _lib.check(self.lib.pearl_sample_rows_multi(
            _lib.ROWS_LOGITS32, _device.ptr(rows_ptrs), n, self.V, _device.ptr(sptrs), U_TABLE, _addr(sptrs, n),
            invt, flags, out_addr, _device.ptr(self.status), _device.stream_ptr(stream)), "pick (batched)")

    def chain_desc(self, r_slot: int, p_addr: int, q_addr: int, drafted: int, tail: int, stride: int, n: int,
                   base: int) -> np.ndarray:
        """One pearl_verify_chain descriptor (include/pearl_b200.h) as 10 int64 words."""
        return np.array([p_addr, q_addr, drafted, tail, int(self.tables[1, r_slot].data_ptr()),
                         _addr(self.cursors[1], r_slot), _addr(self.verdict[r_slot]), _addr(self.work[r_slot]),
                         n | (base << 32), stride], np.int64)

    def verify_multi(self, d: torch.Tensor, n_chains: int, n_clusters: int, invt: float, greedy: bool, bonus: bool,
                     stream) -> None:
        """K1 for every active sequence in one launch (pearl_spec_verify_multi);
        `d` = the uploaded chain_desc words."""
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE | (_lib.F_BONUS if bonus else 0)
        _lib.check(self.lib.pearl_spec_verify_multi(
            _lib.ROWS_LOGITS32, _device.ptr(d), n_chains, n_clusters, self.V, U_TABLE, invt, flags,
            _device.stream_ptr(stream)), "spec_verify_multi (batched)")

    def replay(self, key: tuple, fn, stream) -> None:
        """Run fn(stream) as a CUDA graph keyed by its shape (captured on first use)."""
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn(torch.cuda.current_stream())
            self.graphs[key] = g
        with torch.cuda.stream(stream):
            g.replay()

    def row(self, t: torch.Tensor, r: int) -> int:
        return int(t.data_ptr()) + r * self.V * 4

    def prefill(self, seqs: List[_Seq], stats: dict) -> None:
        """All sequences' prompts (all but the last committed token) into their slots."""
        toks, slots, pos = [], [], []
        for s in seqs:
            body = s.committed[:-1]
            toks += body
            slots += [s.slot] * len(body)
            pos += list(range(len(body)))
        if not toks:
            return
        self.begin_step()
        t, sl, p = self.upload([np.array(toks, np.int32), np.array(slots, np.int32), np.array(pos, np.int32)])
        self.ev[0].record()
        main = torch.cuda.current_stream()
        self.target_stream.wait_stream(main)
        with torch.cuda.stream(self.target_stream):
            self.target.forward_slots(t, len(toks), sl, p, None, self.target_stream)
        if self.draft is not None:  # the two prefills are independent: run them concurrently
            self.draft_stream.wait_stream(main)
            with torch.cuda.stream(self.draft_stream):
                self.draft.forward_slots(t, len(toks), sl, p, None, self.draft_stream)
            main.wait_stream(self.draft_stream)
        main.wait_stream(self.target_stream)
        self.ev[1].record()
        self.ev[1].synchronize()
        dt = self.ev[0].elapsed_time(self.ev[1]) / 1e3
        stats["device_s"] += dt
        stats["prefill_s"] += dt

    def refill(self, seqs: List[_Seq], rngs) -> None:
        """Reload a sequence's table when its cursor nears the end (as fastpath._Tables)."""
        for s in seqs:
            for sel, attr in ((0, "dcur"), (1, "vcur")):
                rng = rngs[s.slot][sel]
                used = getattr(s, attr)
                if rng is not None and used > U_TABLE - (2 * self.g + 8):
                    rng.consume(used)
                    self.load_table(sel, s.slot, rng)
                    self.cursors[sel, s.slot] = 0
                    setattr(s, attr, 0)


def _addr(t: torch.Tensor, i: int = 0) -> int:
    return int(t.data_ptr()) + i * t.element_size()


def _setup(target, draft, prompts, cfg, seeds, kind):
    from .engines import DecodeResult  # noqa: F401
    B = len(prompts)
    if B < 1:
        raise ValueError("need at least one prompt")
    seeds = list(seeds) if seeds is not None else [derive_seed(cfg.seed, i) for i in range(B)]
    if len(seeds) != B:
        raise ValueError("one seed per prompt")
    rt = _runtime(target, draft, B, max(cfg.gamma, 1))
    seqs = [_Seq(i, [target.bos_id] + [int(t) for t in pr], replace(cfg, seed=int(seeds[i])))
            for i, pr in enumerate(prompts)]
    rngs = []
    for s in seqs:
        if s.cfg.greedy:
            rngs.append((None, None))
        elif kind == "ar":
            rngs.append((None, RandomStream(s.cfg.seed)))
        else:
            root = RandomStream(s.cfg.seed)
            rngs.append((root.split(0), root.split(1)))
    rt.cursors.zero_()
    for s in seqs:
        for sel in (0, 1):
            if rngs[s.slot][sel] is not None:
                rt.load_table(sel, s.slot, rngs[s.slot][sel])
        if len(s.committed) + 2 * rt.g + 4 >= rt.max_len:
            raise ValueError("prompt does not fit the KV cache")
    stats = {"device_s": 0.0, "prefill_s": 0.0, "steps": 0, "batch": B}
    return rt, seqs, rngs, stats


def _runtime(target, draft, B, g) -> BatchRuntime:
    cache = target.__dict__.setdefault("_pearl_batch_runtimes", {})
    key = (id(draft), B, g)
    rt = cache.get(key)
    if rt is None:
        rt = BatchRuntime(target, draft, B, g)
        cache[key] = rt
    return rt


def _draft_prepare(rt: BatchRuntime, act: List[_Seq], gamma: int, par: int):
    """Host side of a draft block: catch-up windows, positions and pick-row
    tables, uploaded on the current stream.  Returns (device buffers, q row
    address of x_0 per sequence, catch-up counts)."""
    n = len(act)
    toks, slots, pos, last = [], [], [], []
    m0s = []
    for s in act:
        cu = (s.committed + s.pending)[s.dpos:]
        m0s.append(len(cu))
        toks += cu
        slots += [s.slot] * len(cu)
        pos += list(range(s.dpos, s.dpos + len(cu)))
        last.append(len(toks) - 1)
    slot_arr = np.array([s.slot for s in act], np.int32)
    posj = [np.array([s.dpos + m0s[r] + j - 1 for r, s in enumerate(act)], np.int32) for j in range(1, gamma)]
    rows0 = np.array([rt.row(rt.stage, r) for r in last], np.int64)
    rowsj = [np.array([rt.row(rt.qbuf[par, j], r) for r in range(n)], np.int64) for j in range(1, gamma)]
    B, c0 = rt.B, rt.tcap
    bufs = rt.upload([np.array(toks, np.int32), np.array(slots, np.int32), np.array(pos, np.int32), slot_arr,
                      rows0, rt.stream_ptrs(0, act)] + posj + rowsj,
                     caps=[c0, c0, c0, B, B, 2 * B] + [B] * (gamma - 1) + [B] * (gamma - 1))
    return (bufs, len(toks), par), [rt.row(rt.stage, r) for r in last], m0s


def _draft_launch(rt: BatchRuntime, prep, n: int, gamma: int, par: int, invt: float, greedy: bool, stream) -> None:
    """gamma draft iterations for every active sequence on `stream` (one CUDA
    graph per (catch-up tokens, sequences, gamma, parity)): x_j lands in rt.xs[j, rank]."""
    (bufs, n_tok, par) = prep
    t0, s0, p0, sl, r0, sp = bufs[:6]
    pj = bufs[6:6 + gamma - 1]
    rj = bufs[6 + gamma - 1:]
    d = rt.draft

    def body(st):
        d.forward_slots(t0, n_tok, s0, p0, rt.stage, st)
        rt.pick(r0, n, _addr(rt.xs[0]), sp, invt, greedy, st)
        for j in range(1, gamma):
            d.forward_slots(rt.xs[j - 1], n, sl, pj[j - 1], rt.qbuf[par, j], st)
            rt.pick(rj[j - 1], n, _addr(rt.xs[j]), sp, invt, greedy, st)
    rt.replay(("draft", n_tok, n, gamma, par, invt, greedy), body, stream)


def _read_back(rt: BatchRuntime, n: int, gamma: int) -> tuple:
    B = rt.B
    h = rt.out_host
    h[:B * 8].copy_(rt.verdict.view(-1), non_blocking=True)
    h[B * 8:B * 8 + (rt.g + 1) * B].copy_(rt.xs.view(-1), non_blocking=True)
    c0 = B * 8 + (rt.g + 1) * B
    h[c0:c0 + 2 * B].copy_(rt.cursors.view(-1), non_blocking=True)
    h[c0 + 2 * B:].copy_(rt.status, non_blocking=True)
    rt.ev[1].record()
    rt.ev[1].synchronize()
    a = h.numpy()
    verdict = a[:B * 8].reshape(B, 8)
    xs = a[B * 8:c0].reshape(rt.g + 1, B)
    cur = a[c0:c0 + 2 * B].reshape(2, B)
    _lib.check(int(a[c0 + 2 * B]), "pick (batched)")
    return verdict, xs, cur


def _single(kind: str, draft, target, prompts, cfg, seeds):
    """B == 1: the graph-captured single-sequence engine (same tokens and
    traces by construction; it is the faster implementation of a batch of one)."""
    from . import fastpath
    seed = int(seeds[0]) if seeds is not None else derive_seed(cfg.seed, 0)
    c = replace(cfg, seed=seed)
    if kind == "pearl":
        return [fastpath.decode_pearl(draft, target, prompts[0], c)]
    if kind == "sd":
        return [fastpath.decode_sd(draft, target, prompts[0], c)]
    return [fastpath.decode_autoregressive(target, prompts[0], c)]


def decode_pearl_batch(draft: LlamaModel, target: LlamaModel, prompts: Sequence[Sequence[int]], cfg,
                       seeds: Optional[Sequence[int]] = None) -> list:
    """decode_pearl (engines.py:532-591) for B prompts in lockstep; result i
    equals decode_pearl(draft, target, prompts[i], replace(cfg, seed=seeds[i]))
    (seeds default to the CLI's derive_seed(cfg.seed, i))."""
    from .engines import DecodeResult, StepTrace, finalize_step
    if len(prompts) == 1:
        return _single("pearl", draft, target, prompts, cfg, seeds)
    gamma = cfg.gamma
    rt, seqs, rngs, stats = _setup(target, draft, prompts, cfg, seeds, "pearl")
    invt, greedy = inv_temp(cfg.temperature), bool(cfg.greedy)
    t_d1, t_t = draft.latency.forward_time, target.latency.forward_time
    rt.prefill(seqs, stats)
    par = 0
    while True:
        act = [s for s in seqs if not s.done]
        if not act:
            break
        for s in act:
            if len(s.committed) + len(s.pending) + gamma + 2 >= rt.max_len:
                raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        n = len(act)
        main = torch.cuda.current_stream()
        rt.ev[0].record()
        rt.begin_step()
        # host side first (one staging slab), then fork: target || draft
        ttok, tslot, tpos, offs = [], [], [], []
        for s in act:
            w = [s.committed[-1]] + s.pending
            offs.append(len(ttok))
            ttok += w
            tslot += [s.slot] * len(w)
            tpos += list(range(len(s.committed) - 1, len(s.committed) - 1 + len(w)))
        tt, ts, tp = rt.upload([np.array(ttok, np.int32), np.array(tslot, np.int32), np.array(tpos, np.int32)],
                               caps=[rt.tcap] * 3)
        prep, q0, m0s = _draft_prepare(rt, act, gamma, par)
        ptr_rows = []
        for r, s in enumerate(act):
            k = len(s.pending)
            ptr_rows.append(np.array([rt.row(rt.trows, offs[r] + j) for j in range(k + 1)]
                                     + s.pending_q + [q0[r]], np.int64))
        pend_all = [t for s in act for t in s.pending]
        ptrs, pend = rt.upload([np.concatenate(ptr_rows), np.array(pend_all or [0], np.int32)])
        # chains = pending + [x_0] (x_0 read on the device): one K1 launch for all sequences
        descs, off, poff, base = [], 0, 0, 0
        for r, s in enumerate(act):
            k = len(s.pending)
            pa = _addr(ptrs, off)
            x0 = _addr(rt.xs[0], r)
            descs.append(rt.chain_desc(s.slot, pa, pa + 8 * (k + 1), _addr(pend, poff) if k else x0, x0, 1, k + 1,
                                       base))
            off += 2 * k + 2
            poff += k
            base += k + 1
        (dd,) = rt.upload([np.concatenate(descs)])
        rt.draft_stream.wait_stream(main)
        rt.target_stream.wait_stream(main)
        nt = len(ttok)
        rt.replay(("target", nt), lambda st: target.forward_slots(tt, nt, ts, tp, rt.trows, st), rt.target_stream)
        _draft_launch(rt, prep, n, gamma, par, invt, greedy, rt.draft_stream)
        main.wait_stream(rt.draft_stream)
        main.wait_stream(rt.target_stream)
        rt.verify_multi(dd, n, base, invt, greedy, False, main)
        verdict, xs_h, cur = _read_back(rt, n, gamma)
        stats["device_s"] += rt.ev[0].elapsed_time(rt.ev[1]) / 1e3
        stats["steps"] += 1
        for r, s in enumerate(act):
            v = verdict[s.slot]
            _lib.check(int(v[0]), "decode_pearl_batch step")
            n_acc, corr = int(v[1]), int(v[2])
            xs = [int(xs_h[j, r]) for j in range(gamma)]
            k = len(s.pending)
            chain = s.pending + [xs[0]]
            kind = "pre_verify" if k == 0 and not (s.steps and s.steps[-1].correction is None) else "post_verify"
            if corr < 0:
                s.committed += chain
                s.pending = xs[1:]
                s.pending_q = [rt.row(rt.qbuf[par, j], r) for j in range(1, gamma)]
                acc, cval, delta = k + 1, None, k + 1
            else:
                s.committed += chain[:n_acc] + [corr]
                s.pending, s.pending_q = [], []
                acc, cval, delta = n_acc, corr, n_acc + 1
            s.dpos = min(s.dpos + m0s[r] + gamma - 1, len(s.committed) + len(s.pending) - 1)
            if kind == "pre_verify":
                acc = 1 if corr < 0 else 0
            s.dcur, s.vcur = int(cur[0, s.slot]), int(cur[1, s.slot])
            produced = len(s.committed) - s.n0 - delta
            trace = StepTrace(len(s.steps), kind, tuple(xs), acc, cval, delta, gamma * t_d1, t_t)
            stop = finalize_step(tuple(s.committed), s.n0, produced, s.cfg)
            if stop is not None:
                s.steps.append(replace(trace, finalized_delta=stop - produced))
                s.tokens = tuple(s.committed[s.n0:s.n0 + stop])
                s.done = True
            else:
                s.steps.append(trace)
        rt.refill(act, rngs)
        par ^= 1
    return [DecodeResult(s.tokens, tuple(s.steps), stats=dict(stats)) for s in seqs]


def decode_sd_batch(draft: LlamaModel, target: LlamaModel, prompts: Sequence[Sequence[int]], cfg,
                    seeds: Optional[Sequence[int]] = None) -> list:
    """decode_sd (engines.py:344-394) for B prompts in lockstep."""
    from .engines import DecodeResult, StepTrace
    if len(prompts) == 1:
        return _single("sd", draft, target, prompts, cfg, seeds)
    gamma = cfg.gamma
    rt, seqs, rngs, stats = _setup(target, draft, prompts, cfg, seeds, "sd")
    invt, greedy = inv_temp(cfg.temperature), bool(cfg.greedy)
    t_d, t_t = gamma * draft.latency.forward_time, target.latency.forward_time
    rt.prefill(seqs, stats)
    while True:
        act = [s for s in seqs if not s.done]
        if not act:
            break
        for s in act:
            if len(s.committed) + gamma + 4 >= rt.max_len:
                raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        n = len(act)
        main = torch.cuda.current_stream()
        rt.ev[0].record()
        rt.begin_step()
        # same staging layout as a PEARL step (target region first), so the
        # draft block's captured graph reads the same fixed addresses
        rt.upload([np.zeros(0, np.int32)] * 3, caps=[rt.tcap] * 3)
        prep, q0, m0s = _draft_prepare(rt, act, gamma, 0)
        # target window [committed[-1]] + xs: the ids come from the device picks
        tslot, tpos, offs, first = [], [], [], []
        for r, s in enumerate(act):
            offs.append(len(tslot))
            first.append(s.committed[-1])
            tslot += [s.slot] * (gamma + 1)
            tpos += list(range(len(s.committed) - 1, len(s.committed) + gamma))
        ptr_rows = []
        for r, s in enumerate(act):
            ptr_rows.append(np.array([rt.row(rt.trows, offs[r] + j) for j in range(gamma + 1)]
                                     + [q0[r]] + [rt.row(rt.qbuf[0, j], r) for j in range(1, gamma)], np.int64))
        ts, tp, ff, ptrs = rt.upload([np.array(tslot, np.int32), np.array(tpos, np.int32), np.array(first, np.int32),
                                      np.concatenate(ptr_rows)])
        # chain r = xs[:gamma, r] (stride B in rt.xs), bonus row p_gamma: one K1 launch
        descs, off = [], 0
        for r, s in enumerate(act):
            pa = _addr(ptrs, off)
            descs.append(rt.chain_desc(s.slot, pa, pa + 8 * (gamma + 1), _addr(rt.xs[0], r), 0, rt.B, gamma,
                                       r * (gamma + 1)))
            off += 2 * gamma + 1
        (dd,) = rt.upload([np.concatenate(descs)])
        _draft_launch(rt, prep, n, gamma, 0, invt, greedy, main)
        # window ids: [first_r, xs[0][r], .., xs[gamma-1][r]] per sequence, gathered on the device
        tt = torch.empty((n, gamma + 1), dtype=torch.int32, device=rt.dev)
        tt[:, 0] = ff
        tt[:, 1:] = rt.xs[:gamma, :n].t()
        target.forward_slots(tt.view(-1), n * (gamma + 1), ts, tp, rt.trows, main)
        rt.verify_multi(dd, n, n * (gamma + 1), invt, greedy, True, main)
        verdict, xs_h, cur = _read_back(rt, n, gamma)
        stats["device_s"] += rt.ev[0].elapsed_time(rt.ev[1]) / 1e3
        stats["steps"] += 1
        for r, s in enumerate(act):
            v = verdict[s.slot]
            _lib.check(int(v[0]), "decode_sd_batch step")
            n_acc, corr, bonus = int(v[1]), int(v[2]), int(v[5])
            xs = [int(xs_h[j, r]) for j in range(gamma)]
            block = xs[:n_acc] + [bonus if corr < 0 else corr]
            appended = 0
            for tok in block:
                s.committed.append(tok)
                appended += 1
                if (s.cfg.eos_id is not None and tok == s.cfg.eos_id) or len(s.committed) - s.n0 >= s.cfg.max_new_tokens:
                    s.done = True
                    break
            s.dpos = min(s.dpos + m0s[r] + gamma - 1, len(s.committed) - 1)
            s.dcur, s.vcur = int(cur[0, s.slot]), int(cur[1, s.slot])
            s.steps.append(StepTrace(len(s.steps), "sd", tuple(xs), min(n_acc, appended), None if corr < 0 else corr,
                                     appended, t_d, t_t))
            if s.done:
                s.tokens = tuple(s.committed[s.n0:])
        rt.refill(act, rngs)
    return [DecodeResult(s.tokens, tuple(s.steps), stats=dict(stats)) for s in seqs]


def decode_autoregressive_batch(target: LlamaModel, prompts: Sequence[Sequence[int]], cfg,
                                seeds: Optional[Sequence[int]] = None, block: int = 8) -> list:
    """decode_autoregressive (engines.py:289-319) for B prompts in lockstep:
    `block` steps of (one slot-mode forward over the B last tokens -> B picks)
    per host sync."""
    from .engines import DecodeResult, StepTrace
    if len(prompts) == 1:
        return _single("ar", None, target, prompts, cfg, seeds)
    rt, seqs, rngs, stats = _setup(target, None, prompts, cfg, seeds, "ar")
    invt, greedy = inv_temp(cfg.temperature), bool(cfg.greedy)
    t_t = target.latency.forward_time
    rt.prefill(seqs, stats)
    for s in seqs:
        s.out: List[int] = []
    while True:
        act = [s for s in seqs if not s.done]
        if not act:
            break
        n = len(act)
        G = max(1, min(block, min(s.cfg.max_new_tokens - len(s.out) for s in act)))
        for s in act:
            if len(s.committed) + G + 1 >= rt.max_len:
                raise ValueError("decode exceeds the KV-cache capacity (raise max_seq)")
        main = torch.cuda.current_stream()
        rt.ev[0].record()
        rt.begin_step()
        slot_arr = np.array([s.slot for s in act], np.int32)
        last = np.array([s.committed[-1] for s in act], np.int32)
        posg = [np.array([len(s.committed) - 1 + j for s in act], np.int32) for j in range(G)]
        rows = np.array([rt.row(rt.trows, r) for r in range(n)], np.int64)
        bufs = rt.upload([slot_arr, last, rows, rt.stream_ptrs(1, act)] + posg)
        sl, lt, rp, sp = bufs[:4]
        bufs = bufs[1:]
        toks = torch.empty((G + 1, n), dtype=torch.int32, device=rt.dev)
        toks[0].copy_(lt)
        for j in range(G):
            target.forward_slots(toks[j], n, sl, bufs[3 + j], rt.trows, main)
            rt.pick(rp, n, _addr(toks[j + 1]), sp, invt, greedy, main)
        h = torch.empty((G, n), dtype=torch.int32).pin_memory()
        h.copy_(toks[1:], non_blocking=True)
        cur_h = torch.empty((2, rt.B), dtype=torch.int32).pin_memory()
        cur_h.copy_(rt.cursors, non_blocking=True)
        rt.ev[1].record()
        rt.ev[1].synchronize()
        stats["device_s"] += rt.ev[0].elapsed_time(rt.ev[1]) / 1e3
        stats["steps"] += G
        _lib.check(int(rt.status.item()), "pick (batched)")
        out = h.numpy()
        cur = cur_h.numpy()
        for r, s in enumerate(act):
            for j in range(G):
                tok = int(out[j, r])
                s.committed.append(tok)
                s.out.append(tok)
                s.steps.append(StepTrace(len(s.steps), "ar", (), 0, None, 1, 0.0, t_t))
                if (s.cfg.eos_id is not None and tok == s.cfg.eos_id) or len(s.out) >= s.cfg.max_new_tokens:
                    s.done = True
                    break
            s.vcur = int(cur[1, s.slot])
            if s.done:
                s.tokens = tuple(s.out)
        rt.refill(act, rngs)
    return [DecodeResult(s.tokens, tuple(s.steps), stats=dict(stats)) for s in seqs]
