"""CPU restatement of the reference's distribution arithmetic (TEST ORACLE ONLY).

Follows ``/root/reference/pkg/src/pearl_lab/core.py``:

* ``normalize``   -- ProbDist.__init__ validation + renormalisation + CDF
                     (core.py:83-101; NORM_TOL core.py:21, MAX_VOCAB core.py:24)
* ``sample_index``-- ``sample``: searchsorted(cdf, u, 'right') (core.py:182-190)
* ``residual``    -- ``residual_dist``: norm(max(p - q, 0)) (core.py:193-214)

plus the two pieces of arithmetic the B200 kernels must reproduce bit-for-bit:

* ``pairwise_sum_tree`` -- numpy's pairwise summation tree (the algorithm
  behind ``ndarray.sum()`` for contiguous float64, which ProbDist and
  residual_dist call).  ``np.sum`` is used for speed; the explicit tree is kept
  to pin that the device emulation (csrc/probdist.cuh) follows the same tree.
* ``dev_expf`` / ``logits_to_p1`` -- the *device* definition of a model's
  next-token distribution from fp32 logits (the reference has no neural model,
  so this definition is ours).  It is
  built only from IEEE fp32 mul/add/sub/rint/ldexp so numpy reproduces the
  CUDA result exactly.
"""

from __future__ import annotations

import numpy as np

NORM_TOL = 1e-9          # core.py:21
MAX_VOCAB = 65536        # core.py:24
RESIDUAL_FLOOR = 1e-15   # core.py:211


class OracleInvalidDistribution(ValueError):
    """Mirror of core.InvalidDistribution (core.py:27-28)."""


class OracleAllZeroResidual(ValueError):
    """Mirror of core.AllZeroResidual (core.py:31-32)."""


class OracleZeroDraftProb(ValueError):
    """Mirror of core.ZeroDraftProb (core.py:35-36)."""


# -- numpy pairwise summation, restated ---------------------------------------

_PW_BLOCK = 128  # numpy PW_BLOCKSIZE


def pairwise_sum_tree(a: np.ndarray) -> float:
    """numpy's pairwise sum of a contiguous float64 vector, written out.

    n < 8: sequential from 0.0; 8 <= n <= 128: eight strided accumulators
    combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the n % 8 tail in
    order; n > 128: split at n2 = n//2 - (n//2) % 8 and add the two halves.
    """
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.size
    if n < 8:
        res = 0.0
        for x in a:
            res = float(np.float64(res) + x)
        return res
    if n <= _PW_BLOCK:
        r = [np.float64(a[j]) for j in range(8)]
        stop = n - (n % 8)
        for i in range(8, stop, 8):
            for j in range(8):
                r[j] = r[j] + a[i + j]
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(stop, n):
            res = res + a[i]
        return float(res)
    n2 = n // 2
    n2 -= n2 % 8
    return float(np.float64(pairwise_sum_tree(a[:n2])) + np.float64(pairwise_sum_tree(a[n2:])))


def pairwise_sum(a: np.ndarray) -> float:
    """Fast path: numpy's own reduction (same tree as pairwise_sum_tree)."""
    return float(np.ascontiguousarray(a, dtype=np.float64).sum())


# -- ProbDist semantics -------------------------------------------------------


def normalize(probs, enforce_max_vocab: bool = False):
    """ProbDist.__init__ (core.py:83-101): validate, renormalise, build CDF.

    Returns (probs, cdf) as read-only float64 arrays.  ``enforce_max_vocab``
    reproduces the reference's V <= 65536 limit; the B200 build lifts it
    (Llama-3 V=128256) and the oracle follows the build by default.
    """
    arr = np.asarray(probs, dtype=np.float64)
    if arr.ndim != 1:
        raise OracleInvalidDistribution(f"expected a 1-d vector, got shape {arr.shape}")
    hi = MAX_VOCAB if enforce_max_vocab else np.iinfo(np.int32).max
    if not 2 <= arr.size <= hi:
        raise OracleInvalidDistribution(f"vector length {arr.size} outside [2, {hi}]")
    if not np.all(np.isfinite(arr)):
        raise OracleInvalidDistribution("probabilities must be finite")
    if np.any(arr < 0.0):
        raise OracleInvalidDistribution("negative probability")
    total = pairwise_sum(arr)
    if total == 0.0:
        raise OracleInvalidDistribution("all-zero probability vector")
    if abs(total - 1.0) > NORM_TOL:
        raise OracleInvalidDistribution(f"mass {total!r} is farther than {NORM_TOL} from 1")
    arr = arr / total
    cdf = np.cumsum(arr)          # strictly sequential fp64 accumulation
    cdf[-1] = 1.0                 # top-bin guard (core.py:99)
    arr.flags.writeable = False
    cdf.flags.writeable = False
    return arr, cdf


def sample_index(cdf: np.ndarray, u: float) -> int:
    """``sample`` (core.py:182-190): first index whose CDF strictly exceeds u."""
    return int(np.searchsorted(cdf, u, side="right"))


def sample_index_seq(probs: np.ndarray, u: float) -> int:
    """Same as sample_index but walking the sequential cumsum explicitly.

    Documents the rule the device kernel's exact fallback follows: the
    running fp64 sum c_i = c_{i-1} + a_i, answer = first i with c_i > u, and
    the last bin catches everything (cdf[-1] forced to 1.0).
    """
    c = 0.0
    n = len(probs)
    for i in range(n - 1):
        c = float(np.float64(c) + np.float64(probs[i]))
        if c > u:
            return i
    return n - 1


def residual(p_probs: np.ndarray, q_probs: np.ndarray):
    """``residual_dist`` (core.py:193-214) -> (probs, cdf) of norm(max(p-q, 0))."""
    if p_probs.size != q_probs.size:
        raise OracleInvalidDistribution("vocab mismatch")
    r = np.maximum(p_probs - q_probs, 0.0)
    mass = pairwise_sum(r)
    if mass < RESIDUAL_FLOOR:
        raise OracleAllZeroResidual("target and draft distributions are identical")
    return normalize(r / mass)


# -- device distribution definition (fp32 logits -> fp64 probabilities) ------

LOG2E_F = np.float32(1.4426950408889634)
LN2_HI_F = np.float32(0.693359375)
LN2_LO_F = np.float32(-2.12194440e-4)
EXP_FLUSH_F = np.float32(-80.0)
# Taylor coefficients 1/k! for k = 7..0 (Horner order), fp32.
EXP_POLY_F = tuple(np.float32(c) for c in (
    1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0))


def dev_expf(x: np.ndarray) -> np.ndarray:
    """Bit-exact CPU twin of ``pearl_dev_expf`` in csrc/probdist.cuh.

    Cody-Waite reduction x = k ln2 + r, degree-7 Horner polynomial, scale by
    2**k; every step is a single IEEE fp32 RN operation (no FMA), inputs
    below -80 flush to 0 so every non-zero result is a normal float.
    """
    x = np.asarray(x, dtype=np.float32)
    xc = np.maximum(x, EXP_FLUSH_F)
    t = (xc * LOG2E_F).astype(np.float32)
    k = np.rint(t).astype(np.float32)
    r = (xc - (k * LN2_HI_F).astype(np.float32)).astype(np.float32)
    r = (r - (k * LN2_LO_F).astype(np.float32)).astype(np.float32)
    p = np.full_like(r, EXP_POLY_F[0])
    for c in EXP_POLY_F[1:]:
        p = (p * r).astype(np.float32)
        p = (p + c).astype(np.float32)
    out = np.ldexp(p, k.astype(np.int32)).astype(np.float32)
    return np.where(x < EXP_FLUSH_F, np.float32(0.0), out).astype(np.float32)


def logits_to_p1(logits: np.ndarray, inv_temperature: float = 1.0) -> np.ndarray:
    """The device's next-token law from fp32 logits, as a float64 vector p1.

    p1 = e / S with e_i = dev_expf((l_i - max l) * invT) widened to fp64 and
    S the numpy pairwise sum of e.  ProbDist(p1) then renormalises once more
    exactly like the reference (core.py:91-96).
    """
    l = np.asarray(logits, dtype=np.float32)
    # -inf marks a banned token (probability 0); NaN / +inf are invalid.
    if np.any(np.isnan(l)) or np.any(l == np.inf):
        raise OracleInvalidDistribution("NaN or +inf logits")
    m = l.max()
    if m == -np.inf:
        raise OracleInvalidDistribution("all logits are -inf")
    x = ((l - m).astype(np.float32) * np.float32(inv_temperature)).astype(np.float32)
    e = dev_expf(x).astype(np.float64)
    s = pairwise_sum(e)
    return e / s


def logits_to_probs(logits: np.ndarray, inv_temperature: float = 1.0):
    """(probs, cdf) of ProbDist(logits_to_p1(...))."""
    return normalize(logits_to_p1(logits, inv_temperature))
