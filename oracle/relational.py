"""numpy restatement of the reference's hot-path operators (test infrastructure).

Columns are plain numpy arrays; dictionary columns are int64 code arrays with
the dictionary passed alongside where semantics need it.  References are to
/root/reference/pkg/src/tensorquery (tq/).
"""

from __future__ import annotations

import bisect
from typing import Optional, Sequence

import numpy as np

AVG_STABILIZER = 1e-12  # tq/kernels.py:32
PE_ROW_SUM_TOL = 1e-6  # tq/encodings.py:20

_CMP = {"=": np.equal, "<>": np.not_equal, "<": np.less, ">": np.greater,
        "<=": np.less_equal, ">=": np.greater_equal}


# ---------------------------------------------------------------------------
# filter / compaction
# ---------------------------------------------------------------------------

def comparison_mask(values: np.ndarray, op: str, literal,
                    dictionary: Optional[Sequence[str]] = None) -> np.ndarray:
    """tq/kernels.py:54-84 -- numpy comparison; dictionary literals map to codes,
    an absent literal matches nothing (:74-76)."""
    if dictionary is not None:
        i = bisect.bisect_left(dictionary, literal)
        if i >= len(dictionary) or dictionary[i] != literal:
            return np.zeros(len(values), dtype=bool)
        return _CMP[op](values, i)
    return _CMP[op](values, literal)


def filter_indices(columns: Sequence[np.ndarray], predicates, dictionaries=None) -> np.ndarray:
    """tq/kernels.py:87-96 -- AND of masks, np.nonzero."""
    n = len(columns[0])
    mask = np.ones(n, dtype=bool)
    for idx, op, lit in predicates:
        d = dictionaries.get(idx) if dictionaries else None
        mask &= comparison_mask(columns[idx], op, lit, d)
    return np.nonzero(mask)[0]


def take_rows(values: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """tq/kernels.py:44-51 (gather / fancy-index copy)."""
    return values[indices].copy()


def filter_exact(columns: Sequence[np.ndarray], predicates, dictionaries=None) -> list[np.ndarray]:
    """tq/kernels.py:87-97."""
    if not columns:
        return []
    idx = filter_indices(columns, predicates, dictionaries)
    return [take_rows(c, idx) for c in columns]


def gather_vjp(grad_out: np.ndarray, indices: np.ndarray, src_shape) -> np.ndarray:
    """tq/tensor.py:609-612 -- np.add.at scatter."""
    grad = np.zeros(src_shape, dtype=grad_out.dtype)
    np.add.at(grad, indices, grad_out)
    return grad


# ---------------------------------------------------------------------------
# exact group-by / global aggregate
# ---------------------------------------------------------------------------

def groupby_exact(keys: Sequence[np.ndarray], aggs) -> tuple[list[np.ndarray], list[np.ndarray]]:
    """tq/kernels.py:108-167 -- per-key np.unique, mixed-radix combined id,
    bincount counts, np.add.at sums (float64 accumulator for float input, int64
    for int), avg = float64(sum)/count, occupied groups ascending."""
    n = len(keys[0])
    uniqs, codes = [], []
    for k in keys:
        u, inv = np.unique(k, return_inverse=True)
        uniqs.append(u)
        codes.append(inv.astype(np.int64).reshape(-1))
    spaces = [max(1, len(u)) for u in uniqs]
    combined = np.zeros(n, dtype=np.int64)
    for c, s in zip(codes, spaces):
        combined = combined * s + c
    total = int(np.prod(spaces))
    occupied = np.unique(combined) if n else np.array([], dtype=np.int64)
    counts = np.bincount(combined, minlength=total)[occupied] if n else np.array([], dtype=np.int64)
    out = []
    for func, values in aggs:
        if func == "count":
            out.append(counts.astype(np.int64))
            continue
        if values.dtype.kind == "f":
            sums = np.zeros(total, dtype=np.float64)
        else:
            sums = np.zeros(total, dtype=np.int64)
        np.add.at(sums, combined, values)
        sums = sums[occupied]
        out.append(sums if func == "sum" else sums.astype(np.float64) / counts)
    key_values = []
    rem = occupied.copy()
    for u, s in zip(reversed(uniqs), reversed(spaces)):
        key_values.append(u[rem % s])
        rem //= s
    key_values.reverse()
    return key_values, out


def global_aggregate(row_count: int, aggs) -> list[np.ndarray]:
    """tq/compiler.py:206-215 -- sum keeps the input dtype, avg = mean (NaN if empty)."""
    out = []
    for func, values in aggs:
        if func == "count":
            out.append(np.asarray([row_count], dtype=np.int64))
        elif func == "sum":
            out.append(np.asarray([values.sum()], dtype=values.dtype))
        else:
            out.append(np.asarray([values.mean() if len(values) else np.nan]))
    return out


def dense_exact_counts(codes: Sequence[np.ndarray], spaces: Sequence[int]) -> np.ndarray:
    """tq/kernels.py:238-248."""
    spaces = tuple(int(s) for s in spaces)
    n = len(codes[0]) if codes else 0
    combined = np.zeros(n, dtype=np.int64)
    for c, s in zip(codes, spaces):
        combined = combined * s + c
    return np.bincount(combined, minlength=int(np.prod(spaces))).reshape(spaces)


# ---------------------------------------------------------------------------
# sort / limit
# ---------------------------------------------------------------------------

def stable_order(key: np.ndarray, descending: bool = False) -> np.ndarray:
    """tq/kernels.py:256-264 -- stable argsort of the (negated) key."""
    return np.argsort(-key if descending else key, kind="stable")


def sort_limit(columns, key_index: int, descending=False, limit=None) -> list[np.ndarray]:
    """tq/kernels.py:267-272."""
    order = stable_order(columns[key_index], descending)
    if limit is not None:
        order = order[: max(0, limit)]
    return [c[order].copy() for c in columns]


def limit_rows(columns, count: int) -> list[np.ndarray]:
    """tq/kernels.py:275-280."""
    if not columns:
        return []
    idx = np.arange(min(max(0, count), len(columns[0])))
    return [c[idx].copy() for c in columns]


# ---------------------------------------------------------------------------
# probability encodings and the soft group-by
# ---------------------------------------------------------------------------

def softmax(logits: np.ndarray) -> np.ndarray:
    """tq/tensor.py:515-521 (axis=-1)."""
    shifted = logits - logits.max(axis=-1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=-1, keepdims=True)


def softmax_vjp(probs: np.ndarray, g: np.ndarray) -> np.ndarray:
    """tq/tensor.py:523-525."""
    inner = (g * probs).sum(axis=-1, keepdims=True)
    return probs * (g - inner)


def pe_decode(probs: np.ndarray) -> np.ndarray:
    """tq/encodings.py:161 -- argmax, first maximum wins."""
    return np.argmax(probs, axis=1).astype(np.int64)


def one_hot(codes: np.ndarray, k: int, dtype="float64") -> np.ndarray:
    """tq/encodings.py:175-183."""
    out = np.zeros((len(codes), k), dtype=dtype)
    if len(codes):
        out[np.arange(len(codes)), codes] = 1
    return out


def pe_valid(p: np.ndarray) -> Optional[str]:
    """tq/encodings.py:101-107 -- None if valid, else the failing check."""
    if p.size:
        if p.min() < -PE_ROW_SUM_TOL or p.max() > 1.0 + PE_ROW_SUM_TOL:
            return "range"
        if np.max(np.abs(p.sum(axis=1) - 1.0)) > PE_ROW_SUM_TOL:
            return "rowsum"
    return None


def joint_probabilities(pes: Sequence[np.ndarray]) -> np.ndarray:
    """tq/kernels.py:190-209 -- n x prod(k) joint by broadcast multiplication."""
    n = pes[0].shape[0]
    joint = pes[0]
    for j, p in enumerate(pes[1:], start=1):
        joint = joint.reshape(joint.shape + (1,)) * p.reshape((n,) + (1,) * j + (p.shape[1],))
    return joint


def soft_groupby(pes: Sequence[np.ndarray], agg: str = "count",
                 values: Optional[np.ndarray] = None) -> np.ndarray:
    """tq/kernels.py:212-235 -- dense grid shaped by the key spaces."""
    joint = joint_probabilities(pes)
    counts = joint.sum(axis=0)
    if agg == "count":
        return counts
    n = joint.shape[0]
    w = values if values.dtype.kind == "f" else values.astype(np.float64)
    weighted = (joint * w.reshape((n,) + (1,) * len(pes))).sum(axis=0)
    if agg == "sum":
        return weighted
    return weighted / (counts + AVG_STABILIZER)


def soft_groupby_vjp(pes: Sequence[np.ndarray], grid_grad: np.ndarray,
                     values: Optional[np.ndarray] = None) -> tuple[list[np.ndarray], Optional[np.ndarray]]:
    """VJP of the count / weighted-sum grid w.r.t. each P_j and the values.

    The reference obtains it from its tape (reduce_sum :474 -> mul :364-365 ->
    reshape :544); restated in closed form:
      dP_j[i, c] = sum_{cells, c_j = c} G[cell] w_i prod_{l != j} P_l[i, c_l]
      dw_i       = sum_cells G[cell] prod_l P_l[i, c_l]
    """
    n = pes[0].shape[0]
    m = len(pes)
    w = np.ones(n) if values is None else values.astype(np.float64)
    joint = joint_probabilities(pes)
    grads = []
    letters = "abcdefgh"[:m]
    for j in range(m):
        others = [pes[l] if l != j else np.ones_like(pes[j]) for l in range(m)]
        ops = ",".join("z" + letters[l] for l in range(m))
        prod = np.einsum(f"{ops}->z{letters}", *others)
        g = np.einsum(f"z{letters},{letters}->z{letters[j]}", prod, grid_grad) * w[:, None]
        grads.append(g)
    dw = np.einsum(f"z{letters},{letters}->z", joint, grid_grad)
    return grads, (dw if values is not None else None)


def llp_forward_backward(X: np.ndarray, bag: np.ndarray, W: np.ndarray, b: np.ndarray,
                         target: np.ndarray, bags: int):
    """One trainable LLP query step (SURVEY Appendix A llp TVF) in closed form:
    Linear -> softmax (tq/tensor.py:515) -> soft group-by-count over
    (one-hot bag, PE pred) (tq/kernels.py:212-223) -> MSE (tq/training.py:68-73)
    and the gradient w.r.t. W, b that the reference's tape produces.
    Returns (loss, grid[bags*k], dW, db)."""
    logits = X @ W + b
    P = softmax(logits)
    k = P.shape[1]
    grid = np.zeros((bags, k), dtype=np.result_type(P.dtype, np.float64))
    np.add.at(grid, bag, P)
    g = grid.reshape(-1)
    diff = g - target
    loss = float(np.mean(diff * diff))
    dgrid = (2.0 * diff / diff.size).reshape(bags, k)
    dP = dgrid[bag]
    dZ = softmax_vjp(P, dP)
    return loss, g, X.T @ dZ, dZ.sum(axis=0)


# ---------------------------------------------------------------------------
# equi-join (builder-defined: the reference has none)
# ---------------------------------------------------------------------------

def join_inner(probe: np.ndarray, build: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Sort the build keys (stable), searchsorted each probe key; pairs ordered
    by probe row then ascending build row.  PARITY UNPINNED (no reference)."""
    order = np.argsort(build, kind="stable")
    sk = build[order]
    lo = np.searchsorted(sk, probe, side="left")
    hi = np.searchsorted(sk, probe, side="right")
    cnt = hi - lo
    pi = np.repeat(np.arange(len(probe), dtype=np.int64), cnt)
    starts = np.repeat(lo - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) if len(pi) else lo[:0]
    bi = order[np.arange(len(pi)) + starts] if len(pi) else np.array([], dtype=np.int64)
    return pi, bi.astype(np.int64)


def join_nested_loop(probe: np.ndarray, build: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Brute-force check of join_inner for small inputs."""
    pairs = [(i, j) for i in range(len(probe)) for j in range(len(build)) if probe[i] == build[j]]
    if not pairs:
        return np.array([], dtype=np.int64), np.array([], dtype=np.int64)
    a = np.array(pairs, dtype=np.int64)
    return a[:, 0], a[:, 1]


# ---------------------------------------------------------------------------
# gradient paths: gather VJP and the trainable global aggregates
# ---------------------------------------------------------------------------

def gather_rows_vjp(src_shape, idx: np.ndarray, g: np.ndarray) -> np.ndarray:
    """tq/tensor.py:609-612 -- VJP of an axis-0 gather: zeros of the source
    shape, np.add.at of the upstream rows (duplicate indices accumulate)."""
    grad = np.zeros(src_shape, dtype=g.dtype)
    np.add.at(grad, idx, g)
    return grad


def score_global_soft(X: np.ndarray, W: np.ndarray, b: np.ndarray, threshold, G: np.ndarray):
    """Forward + parameter gradients of ``SELECT SUM(s), AVG(s), COUNT(*) FROM
    (SELECT s FROM lin(T) [WHERE s > threshold])`` in trainable mode, with the
    loss G[0]*SUM + G[1]*AVG: the tape chain Linear -> filter_exact/take_rows
    (gather, VJP gather_rows_vjp) -> GlobalAggSoftOp (tq/compiler.py:265-288:
    reduce_sum, reduce_mean, COUNT a float constant).  threshold None: no WHERE."""
    s = (X @ W + b).reshape(-1)
    idx = np.nonzero(s > threshold)[0] if threshold is not None else np.arange(len(s))
    kept = s[idx]
    m = len(kept)
    total = kept.sum()
    avg = kept.mean() if m else np.nan
    ds_kept = np.full(m, G[0] + (G[1] / m if m else 0.0))
    ds = gather_rows_vjp((len(s),), idx, ds_kept)
    dW = X.T @ ds.reshape(-1, 1)
    db = np.array([ds.sum()])
    return np.array([total]), np.array([avg]), np.array([float(m)]), dW, db
