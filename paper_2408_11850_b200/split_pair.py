r"""Split pair: PEARL with the draft and the target on different GPUs.

The reference overlaps the two phases of a step with a 2-thread
``_PhaseRunner`` (engines.py:241-262) and meets in one host thread to verify.
Here the two phases run on two GPUs, one process each (torchrun ranks), and
meet on the target GPU through K6 (csrc/exchange.cu):

    draft rank (GPU d)                       target rank (GPU t)
    assemble draft catch-up                  assemble window [committed[-1]] + pending
    gamma x (draft forward -> pick)          target forward over the window (M = k+1)
    K6 push: xs + gamma q rows ---NVLink---> mailbox(t)
                                             K6 wait, chain = pending + [xs0]
                                             K1 verify, commit (K5 rollback)
    mailbox(d) <---NVLink--- 32 B verdict    K6 push: verdict
    K6 wait, commit (same verdict)
    D2H summary                              D2H summary

Each rank's step is ONE CUDA graph; the mailboxes are plain device buffers
mapped into the peer process with CUDA IPC, written by the sender's kernel
and polled by a one-thread acquire loop on the receiver, so no host thread
and no NCCL call sits between the phases.  Both ranks run the same
deterministic commit on the same verdict, so their DecodeState mirrors stay
identical (each advances only its own KV cache and uniform cursor), and both
return the same DecodeResult.  Greedy decodes send only the ids (K1's greedy
rule never reads q, engines.py:220-226).

Public API: the reference's ``decode_pearl(draft, target, prefix, cfg)``
with the remote half given as a :class:`PeerModel`::

    # rank 0 (target GPU)                    # rank 1 (draft GPU)
    link = SplitLink.connect(...)            link = SplitLink.connect(...)
    decode_pearl(PeerModel(link), target,    decode_pearl(draft, PeerModel(link),
                 prefix, cfg)                             prefix, cfg)

Adaptive gamma works unchanged: the two ranks exchange their calibrations
once when the link connects, so both planners make the same choices.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import replace
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _device, _lib
from .core import RandomStream
from .errors import DeviceError
from .llama import LlamaModel, inv_temp
from .models import LatencyProfile, SequenceModel

ROLE_TARGET = "target"
ROLE_DRAFT = "draft"

DEFAULT_TIMEOUT_S = 120.0


class SplitLink:
    """K6 mailboxes and sequence counters of one draft<->target link.

    The target rank owns a mailbox for gamma_max q rows + ids; the draft
    rank owns a verdict mailbox.  Each is exported with CUDA IPC and the
    handles (plus both models' calibrations) are exchanged once over
    ``torch.distributed`` (any backend that carries objects: gloo or nccl).
    """

    def __init__(self, role: str, peer_rank: int, vocab: int, gamma_max: int, box: int, peer_box: int,
                 peer_info: dict, timeout_s: float):
        self.role, self.peer_rank, self.V, self.gmax = role, int(peer_rank), int(vocab), int(gamma_max)
        self.box, self.peer_box = box, peer_box
        self.peer_info = peer_info
        self.timeout_ns = int(timeout_s * 1e9)
        dev = torch.device("cuda", torch.cuda.current_device())
        # send_seq, recv_seq (uint64 as int64), arrive (uint32 in an int64 slot)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)  # send, recv, arrive, staging
        # K6 transport: direct peer stores when this GPU can map the peer's
        # memory (NVLink / NVSwitch, or the same device), else copy-engine pushes
        self.mode = "peer_store"
        self.closed = False

    @classmethod
    def connect(cls, role: str, peer_rank: int, vocab: int, gamma_max: int, local_info: dict,
                group=None, timeout_s: float = DEFAULT_TIMEOUT_S) -> "SplitLink":
        """Collective over ``group`` (default WORLD): every rank of the group
        calls it once; each link uses its peer's entry.  ``local_info`` is
        this rank's calibration (``SplitLink.calibrate``)."""
        import torch.distributed as dist
        if role not in (ROLE_TARGET, ROLE_DRAFT):
            raise ValueError("role must be 'target' or 'draft'")
        if not 1 <= gamma_max <= _lib.MAILBOX_MAX_IDS:
            raise ValueError("gamma_max out of range")
        _device.require_cuda()
        lib = _lib.load()
        rows = gamma_max if role == ROLE_TARGET else 0
        nbytes = int(lib.pearl_mailbox_bytes(rows, int(vocab)))
        p = ctypes.c_void_p()
        _lib.check(lib.pearl_mailbox_alloc(nbytes, ctypes.byref(p)), "pearl_mailbox_alloc")
        handle = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        _lib.check(lib.pearl_ipc_export(p, handle), "pearl_ipc_export")
        bus = ctypes.create_string_buffer(64)
        _lib.check(lib.pearl_pci_bus_id(bus, 64), "pearl_pci_bus_id")
        entry = {"role": role, "rank": dist.get_rank(), "handle": handle.raw, "vocab": int(vocab),
                 "gamma_max": int(gamma_max), "info": dict(local_info), "pci": bus.value.decode()}
        peer = exchange_entries(entry, peer_rank, group)
        storable = int(lib.pearl_peer_storable(peer["pci"].encode()))
        if storable < 0:
            _lib.check(storable, "pearl_peer_storable")
        q = ctypes.c_void_p()
        hbuf = ctypes.create_string_buffer(peer["handle"], _lib.IPC_HANDLE_BYTES)
        _lib.check(lib.pearl_ipc_import(hbuf, ctypes.byref(q)), "pearl_ipc_import")
        link = cls(role, peer_rank, vocab, gamma_max, p.value, q.value, peer["info"], timeout_s)
        if storable == 0 or os.environ.get("PEARL_K6_COPY", "0") == "1":
            link.mode = "copy_engine"
        # both sides have mapped each other's mailbox before the first push
        dist.barrier(group=group)
        return link

    @staticmethod
    def calibrate(model: LlamaModel, role: str) -> dict:
        """Forward times the planner needs, measured on this rank's GPU alone."""
        if role == ROLE_DRAFT:
            return {"t_d": model.measure_forward_time(1) + 6e-6, "latency": model.latency.forward_time}
        return {"t_t": {m: model.measure_forward_time(m) for m in (1, 8, 16, 32)},
                "latency": model.latency.forward_time}

    # -- kernel launches (graph-capturable) ---------------------------------
    def _ctr(self, i: int) -> int:
        return int(self.counters.data_ptr()) + 8 * i

    def send(self, ids_addr: int, n_ids: int, rows_addr: Optional[int], n_rows: int, stream) -> None:
        a = _XferArgs(self.peer_box, ids_addr, int(n_ids), rows_addr, int(n_rows), self.V, self._ctr(0),
                      self._ctr(2))
        if self.mode == "copy_engine":
            _lib.check(_lib.load().pearl_xfer_send_copy(ctypes.byref(a), self._ctr(3), _device.stream_ptr(stream)),
                       "pearl_xfer_send_copy")
            return
        _lib.check(_lib.load().pearl_xfer_send(ctypes.byref(a), _device.stream_ptr(stream)), "pearl_xfer_send")

    def wait(self, dst_addr: Optional[int], n_ids: int, status_addr: int, stream) -> None:
        _lib.check(_lib.load().pearl_xfer_wait(self.box, self._ctr(1), dst_addr, int(n_ids), status_addr,
                                               self.timeout_ns, _device.stream_ptr(stream)), "pearl_xfer_wait")

    def rows_addr(self) -> int:
        """Device address of the q rows in this rank's mailbox (target rank)."""
        return int(self.box) + _lib.MAILBOX_ROWS_OFFSET

    def close(self) -> None:
        if self.closed:
            return
        self.closed = True
        lib = _lib.load()
        torch.cuda.synchronize()
        lib.pearl_ipc_close(ctypes.c_void_p(self.peer_box))
        lib.pearl_mailbox_free(ctypes.c_void_p(self.box))


def exchange_entries(entry: dict, peer_rank: int, group=None) -> dict:
    """Link handshake (host side, any torch.distributed backend): every rank
    of ``group`` contributes its entry (role, IPC handle, vocab, gamma_max,
    calibration); returns the peer's entry after checking the two match."""
    import torch.distributed as dist
    allv: List[Optional[dict]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, entry, group=group)
    peer = next((e for e in allv if e is not None and e["rank"] == peer_rank), None)
    if peer is None:
        raise ValueError(f"rank {peer_rank} is not in the link group")
    check_peer(entry, peer)
    return peer


def pair_roles(rank: int, world_size: int) -> tuple:
    """(role, peer rank) of a rank when world_size GPUs form world_size/2
    split pairs: even ranks host targets, odd ranks their drafts."""
    if world_size < 2 or world_size % 2:
        raise ValueError("split pairs need an even number of ranks")
    return (ROLE_TARGET, rank + 1) if rank % 2 == 0 else (ROLE_DRAFT, rank - 1)


def check_peer(mine: dict, peer: dict) -> None:
    """Handshake checks: complementary roles, same vocabulary and gamma_max."""
    if {mine["role"], peer["role"]} != {ROLE_TARGET, ROLE_DRAFT}:
        raise ValueError(f"split pair needs one target and one draft rank, got {mine['role']}/{peer['role']}")
    if mine["vocab"] != peer["vocab"]:
        raise ValueError("draft and target must share a vocabulary")
    if mine["gamma_max"] != peer["gamma_max"]:
        raise ValueError("both ranks of a split pair must use the same gamma_max")


class _XferArgs(ctypes.Structure):
    _fields_ = [("peer_box", ctypes.c_void_p), ("ids", ctypes.c_void_p), ("n_ids", ctypes.c_int32),
                ("rows", ctypes.c_void_p), ("n_rows", ctypes.c_int32), ("V", ctypes.c_int32),
                ("send_seq", ctypes.c_void_p), ("arrive", ctypes.c_void_p)]


class PeerModel(SequenceModel):
    """Stand-in for the half of a split pair that lives on the peer rank.

    Passed to ``decode_pearl`` in place of the remote model.  It has the
    SequenceModel attributes (``vocab_size``, ``latency``) but no local
    forward: the remote model is only reachable through the link."""

    _pearl_peer_model = True

    def __init__(self, link: SplitLink):
        self.link = link
        self.vocab_size = link.V
        self.latency = LatencyProfile(float(link.peer_info.get("latency", 0.0)))

    def next_dist(self, prefix):
        raise DeviceError(f"this model lives on rank {self.link.peer_rank}; "
                          "run decode_pearl with the local half on each rank")


def is_peer_model(m) -> bool:
    return bool(getattr(m, "_pearl_peer_model", False))


# state fields / summary layout shared with fastpath (engine.cu)
from .fastpath import (S_DCUR, S_DPOS, S_TPOS, S_VCUR, SUM_ACCEPTED, SUM_COMMITTED, SUM_CORRECTION,  # noqa: E402
                       SUM_DCUR, SUM_DPOS, SUM_FALLBACK, SUM_HDR, SUM_STATUS, SUM_VCUR, U_TABLE, _CommitArgs,
                       _GammaPlanner, _addr, _FWD_ADVANCE, _FWD_LAST, _new_stats, _Tables, steps_mode_post)


class SplitRuntime:
    """Buffers and step graphs of one rank of a split pair."""

    def __init__(self, model: LlamaModel, link: SplitLink):
        self.model, self.link = model, link
        self.role = link.role
        self.dev = model.device
        V = model.cfg.vocab
        if V != link.V:
            raise ValueError("model vocabulary does not match the link")
        self.V, self.gmax = V, link.gmax
        self.max_len = model.max_seq
        g = self.gmax
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.state = torch.zeros(8, **i32)
        self.seq = torch.zeros(self.max_len + 2 * g + 4, **i32)
        self.pending_tok = torch.zeros(g + 1, **i32)
        self.chain = torch.zeros(2 * g + 2, **i32)
        self.verdict = torch.zeros(8, **i32)
        self.summary = torch.zeros(SUM_HDR + g + 8, **i32)
        self.summary_host = torch.zeros(SUM_HDR + g + 8, dtype=torch.int32).pin_memory()
        self.link_status = torch.zeros(1, **i32)
        self.link_status_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.lib = _lib.load()
        wb = int(self.lib.pearl_verify_work_bytes(g + 2))
        if self.role == ROLE_DRAFT:
            self.draft_in = torch.zeros(g + 4, **i32)
            self.draft_cnt = torch.zeros(1, **i32)
            self.draft_rows = torch.zeros(g + 1, V, dtype=torch.float32, device=self.dev)
            self.draft_row_ptrs = _device.row_ptrs([self.draft_rows[j] for j in range(g + 1)], self.dev)
            self.u_draft = torch.zeros(U_TABLE, dtype=torch.float64, device=self.dev)
            self.work_s = torch.zeros(wb, dtype=torch.uint8, device=self.dev)
            self.sample_status = torch.zeros(1, **i32)
        else:
            self.target_in = torch.zeros(g + 2, **i32)
            self.target_rows = torch.zeros(g + 2, V, dtype=torch.float32, device=self.dev)
            self.target_row_ptrs = _device.row_ptrs([self.target_rows[j] for j in range(g + 2)], self.dev)
            self.pending_rows = torch.zeros(g + 1, V, dtype=torch.float32, device=self.dev)
            box_rows = link.rows_addr()
            # q rows of a chain of k pending + 1 fresh: pending_rows[0..k-1], then the mailbox's row 0
            self.q_row_ptrs = {k: torch.tensor([_addr(self.pending_rows, j * V) for j in range(k)] + [box_rows],
                                               dtype=torch.int64, device=self.dev) for k in range(g + 1)}
            self.box_rows = box_rows
            self.u_verify = torch.zeros(U_TABLE, dtype=torch.float64, device=self.dev)
            self.work_v = torch.zeros(wb, dtype=torch.uint8, device=self.dev)
        self.graphs: Dict[tuple, torch.cuda.CUDAGraph] = {}
        self.graph_launches: Dict[tuple, int] = {}
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        _lib.prepare_vocab(V)

    def _sp(self, field: int) -> int:
        return _addr(self.state, field)

    # -- step bodies ----------------------------------------------------------
    def _commit(self, k: int, gamma: int, draft_rows: Optional[int], pending_rows: Optional[int], stream) -> None:
        a = _CommitArgs(self._sp(0), _device.ptr(self.seq), self.max_len, _device.ptr(self.chain), k, gamma,
                        _device.ptr(self.verdict), _device.ptr(self.pending_tok), pending_rows, draft_rows, self.V, 0,
                        _device.ptr(self.summary))
        _lib.check(self.lib.pearl_pearl_commit(ctypes.byref(a), _device.stream_ptr(stream)), "commit")

    def _draft_body(self, k: int, gamma: int, m0: int, invt: float, greedy: bool) -> None:
        s0 = torch.cuda.current_stream()
        lib, m = self.lib, self.model
        _lib.check(lib.pearl_step_assemble(self._sp(0), _device.ptr(self.seq), _device.ptr(self.pending_tok), None,
                                           _device.ptr(self.draft_in), _device.ptr(self.draft_cnt),
                                           _device.stream_ptr(s0)), "assemble")
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE
        for j in range(gamma):
            tok = _device.ptr(self.draft_in) if j == 0 else _addr(self.chain, k + j - 1)
            _lib.check(lib.pearl_llama_forward(m.handle, tok, m0 if j == 0 else 1, self._sp(S_DPOS),
                                               _FWD_ADVANCE | _FWD_LAST, _addr(self.draft_rows, j * self.V),
                                               _device.stream_ptr(s0)), "draft forward")
            _lib.check(lib.pearl_sample_rows(_lib.ROWS_LOGITS32, _addr(self.draft_row_ptrs, j), 1, self.V,
                                             _device.ptr(self.u_draft), U_TABLE, self._sp(S_DCUR), invt, flags,
                                             _addr(self.chain, k + j), None, _device.ptr(self.sample_status),
                                             _device.ptr(self.work_s), _device.stream_ptr(s0)), "pick")
        # K6 push: xs (+ q rows unless greedy) into the target GPU's mailbox
        self.link.send(_addr(self.chain, k), gamma, None if greedy else _device.ptr(self.draft_rows),
                       0 if greedy else gamma, s0)
        self.link.wait(_device.ptr(self.verdict), 8, _device.ptr(self.link_status), s0)
        if k > 0:
            self.chain[:k].copy_(self.pending_tok[:k])
        self._commit(k, gamma, None, None, s0)
        self.summary_host.copy_(self.summary, non_blocking=True)
        self.link_status_host.copy_(self.link_status, non_blocking=True)

    def _target_body(self, k: int, gamma: int, invt: float, greedy: bool) -> None:
        s0 = torch.cuda.current_stream()
        lib, m = self.lib, self.model
        _lib.check(lib.pearl_step_assemble(self._sp(0), _device.ptr(self.seq), _device.ptr(self.pending_tok),
                                           _device.ptr(self.target_in), None, None, _device.stream_ptr(s0)),
                   "assemble")
        _lib.check(lib.pearl_llama_forward(m.handle, _device.ptr(self.target_in), k + 1, self._sp(S_TPOS), 0,
                                           _device.ptr(self.target_rows), _device.stream_ptr(s0)), "target forward")
        # K6 wait: the draft's xs land in chain[k:], its q rows stay in the mailbox
        self.link.wait(_addr(self.chain, k), gamma, _device.ptr(self.link_status), s0)
        if k > 0:
            self.chain[:k].copy_(self.pending_tok[:k])
        flags = (_lib.F_GREEDY if greedy else 0) | _lib.F_ADVANCE
        _lib.check(lib.pearl_spec_verify(_lib.ROWS_LOGITS32, _device.ptr(self.target_row_ptrs),
                                         _device.ptr(self.q_row_ptrs[k]), _device.ptr(self.chain), k + 1, self.V,
                                         _device.ptr(self.u_verify), U_TABLE, self._sp(S_VCUR), invt, flags,
                                         _device.ptr(self.verdict), None, _device.ptr(self.work_v),
                                         _device.stream_ptr(s0)), "spec_verify")
        self._commit(k, gamma, self.box_rows, _device.ptr(self.pending_rows), s0)
        # K6 push: the 32-byte verdict into the draft GPU's mailbox
        self.link.send(_device.ptr(self.verdict), 8, None, 0, s0)
        self.summary_host.copy_(self.summary, non_blocking=True)
        self.link_status_host.copy_(self.link_status, non_blocking=True)

    def body(self, k: int, gamma: int, m0: int, invt: float, greedy: bool):
        if self.role == ROLE_DRAFT:
            return lambda: self._draft_body(k, gamma, m0, invt, greedy)
        return lambda: self._target_body(k, gamma, invt, greedy)

    def key(self, k: int, gamma: int, m0: int, invt: float, greedy: bool) -> tuple:
        # the target's graph does not depend on the draft catch-up length
        return (k, gamma, m0 if self.role == ROLE_DRAFT else 0, greedy, invt)

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

    def replay(self, key: tuple, body, stats: dict) -> None:
        g = self.graph(key, body)
        self.ev[0].record()
        g.replay()
        self.ev[1].record()
        self.ev[1].synchronize()
        if int(self.link_status_host[0]) != 0:
            _lib.check(int(self.link_status_host[0]), "split-pair exchange")
        stats["device_s"] += self.ev[0].elapsed_time(self.ev[1]) / 1e3
        stats["launches"] += self.graph_launches[key]
        stats["replays"] += 1

    def reset(self, seq0: List[int], stats: dict) -> None:
        C = len(seq0)
        if C + 2 > self.max_len:
            raise ValueError("prompt does not fit the KV cache")
        c0 = int(self.lib.pearl_launch_count())
        self.ev[2].record()
        self.seq[:C].copy_(torch.tensor(seq0, dtype=torch.int32))
        self.state.copy_(torch.tensor([C, 0, 0, 0, 0, 0, 0, 0], dtype=torch.int32))
        self.link_status.zero_()
        if C > 1:
            field = S_DPOS if self.role == ROLE_DRAFT else S_TPOS
            self.model.forward(self.seq[:C - 1], C - 1, self.state[field:field + 1], _FWD_ADVANCE, None)
        self.ev[3].record()
        self.ev[3].synchronize()
        t = self.ev[2].elapsed_time(self.ev[3]) / 1e3
        stats["device_s"] += t
        stats["prefill_s"] += t
        stats["launches"] += int(self.lib.pearl_launch_count()) - c0
        self.model.reset_adapter()

    def load_uniforms(self, table: torch.Tensor, rng: RandomStream) -> None:
        table.copy_(torch.from_numpy(np.array(rng.peek(U_TABLE))))


def _split_runtime(model: LlamaModel, link: SplitLink) -> SplitRuntime:
    cache = model.__dict__.setdefault("_pearl_split_runtimes", {})
    rt = cache.get(id(link))
    if rt is None:
        rt = SplitRuntime(model, link)
        cache[id(link)] = rt
    return rt


class _PlannerFromLink(_GammaPlanner):
    """The adaptive-gamma planner with the calibration both ranks share."""

    def __init__(self, link: SplitLink, local_info: dict, gamma_max: int, gamma0: int):
        d = local_info if link.role == ROLE_DRAFT else link.peer_info
        t = local_info if link.role == ROLE_TARGET else link.peer_info
        self.t_d = float(d["t_d"])
        self.t_t = {int(m): float(v) for m, v in t["t_t"].items()}
        self.meas = {}  # never fed: both ranks price steps with the shared model only
        self.frozen = False
        self.gmax = gamma_max
        self.acc, self.exam = 3.0, 4.0
        self.gamma = gamma0
        self.started = False


def decode_pearl_split(draft, target, prefix: Sequence[int], cfg):
    """decode_pearl (engines.py:532-591) for one rank of a split pair."""
    from .engines import DecodeResult, StepTrace, finalize_step
    if is_peer_model(draft) and not is_peer_model(target):
        model, link = target, draft.link
    elif is_peer_model(target) and not is_peer_model(draft):
        model, link = draft, target.link
    else:
        raise ValueError("exactly one of draft / target must be a PeerModel")
    if link.role != (ROLE_TARGET if model is target else ROLE_DRAFT):
        raise ValueError("the local model's role does not match the link")
    if cfg.gamma > link.gmax or (cfg.adaptive_gamma and cfg.gamma_max > link.gmax):
        raise ValueError("gamma exceeds the link's gamma_max")
    local_info = model.__dict__.get("_pearl_split_calib")
    if local_info is None:
        raise ValueError("calibrate the local model with SplitLink.calibrate before connecting")
    planner = _PlannerFromLink(link, local_info, cfg.gamma_max, cfg.gamma) if cfg.adaptive_gamma else None
    gamma = planner.next_gamma() if planner else cfg.gamma
    dinfo = local_info if link.role == ROLE_DRAFT else link.peer_info
    tinfo = local_info if link.role == ROLE_TARGET else link.peer_info
    t_d1, t_t = float(dinfo["latency"]), float(tinfo["latency"])
    rt = _split_runtime(model, link)
    seq0 = [model.bos_id] + [int(t) for t in prefix]
    n0 = len(seq0)
    stats = _new_stats(gamma=gamma, gammas=[], role=link.role)
    rt.reset(seq0, stats)
    root = RandomStream(cfg.seed)
    if link.role == ROLE_DRAFT:
        tab = _Tables(rt, rt.u_draft, None if cfg.greedy else root.split(0), S_DCUR)
    else:
        tab = _Tables(rt, rt.u_verify, None if cfg.greedy else root.split(1), S_VCUR)
    invt = inv_temp(cfg.temperature)
    greedy = bool(cfg.greedy)
    _precapture(rt, planner, gamma, invt, greedy)
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
        rt.replay(rt.key(k, gamma, m0, invt, greedy), rt.body(k, gamma, m0, invt, greedy), stats)
        s = rt.summary_host.numpy()
        _lib.check(int(s[SUM_STATUS]), "decode_pearl step")
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
        if link.role == ROLE_DRAFT:
            dpos = int(s[SUM_DPOS])
        else:
            dpos = len(committed) + len(pending) - 1  # unused by the target's graphs
        assert int(s[SUM_COMMITTED]) == len(committed)
        if kind == "pre_verify":
            acc = 1 if corr < 0 else 0
        trace = StepTrace(len(steps), kind, tuple(xs), acc, cval, delta, gamma * t_d1, t_t)
        if planner is not None:
            planner.observe(acc, 0 if cval is None else 1)
            gamma = planner.next_gamma()
        field = SUM_DCUR if link.role == ROLE_DRAFT else SUM_VCUR
        tab.advance(int(s[field]), 2 * link.gmax + 8)
        stop = finalize_step(tuple(committed), n0, produced, cfg)
        if stop is not None:
            steps.append(replace(trace, finalized_delta=stop - produced))
            return DecodeResult(tuple(committed[n0:n0 + stop]), tuple(steps), stats=stats)
        steps.append(trace)
        produced = len(committed) - n0
    return DecodeResult(tuple(committed[n0:]), tuple(steps), stats=stats)


def _precapture(rt: SplitRuntime, planner, gamma: int, invt: float, greedy: bool) -> None:
    """Capture the step graphs the decode can reach (fastpath._precapture_pearl)."""
    gammas = planner.candidates() if planner is not None else [gamma]
    for g in gammas:
        prevs = planner.neighbors(g) if planner is not None else [g]
        for k in sorted({0} | {gp - 1 for gp in prevs if gp > 1}):
            rt.graph(rt.key(k, g, 1, invt, greedy), rt.body(k, g, 1, invt, greedy))


def connect_pair(model: LlamaModel, role: str, peer_rank: int, gamma_max: int, group=None,
                 timeout_s: float = DEFAULT_TIMEOUT_S) -> PeerModel:
    """Calibrate the local model, connect the link (collective over ``group``)
    and return the PeerModel standing in for the remote half."""
    info = SplitLink.calibrate(model, role)
    model.__dict__["_pearl_split_calib"] = info
    link = SplitLink.connect(role, peer_rank, model.cfg.vocab, gamma_max, info, group=group, timeout_s=timeout_s)
    return PeerModel(link)
