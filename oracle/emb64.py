"""TEST INFRASTRUCTURE ONLY — an fp64 EmbeddingBag oracle that does NOT follow
the kernels' reduction order.

The reference has no EmbeddingBag (the paper ran FBGEMM,
PAPER.md:64, which is not vendored), so the operator is pinned to its
definition:

* forward: pooled[b, col_t : col_t + D_t] = sum of the rows of
  table t looked up by bag (t, b); an empty bag pools to the zero vector;
* backward: the per-row gradient g_r = sum of grad_pooled[b, col_t:] over
  every lookup of row r (a row looked up k times in one bag counts k times);
* row-wise SGD: w_r <- w_r - lr * g_r;
* exact row-wise Adagrad (FBGEMM's ``EXACT_ROWWISE_ADAGRAD``, one fp32 state
  per row): m_r <- m_r + mean_k(g_rk^2); w_r <- w_r - lr * g_r / (sqrt(m_r) + eps).

Everything is accumulated in float64 (torch CPU ``index_add_``, any order), so
the result is the exact value to ~1e-15; ``bound_*`` return the floating-point
error budget the fp32 kernels must meet: 1e-5 relative to the condition of
each sum (sum of |terms|), the tolerance BASELINE.json's north_star states
("within 1e-5 relative in fp32").  Weights come from ``oracle.C().init_table``
(the deterministic init the operator also uses, or_init_weight).
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-5


def _bags(offsets, t, B):
    o = np.asarray(offsets[t * B:(t + 1) * B + 1], np.int64)
    lens = np.diff(o)
    return int(o[0]), int(o[-1]), np.repeat(np.arange(B, dtype=np.int64), lens)


def forward(B, dims, offsets, indices, weights):
    """Returns (pooled fp64 [B, sum D], abs_sum fp64 [B, sum D])."""
    import torch

    T = len(dims)
    out = torch.zeros(B, int(sum(dims)), dtype=torch.float64)
    aout = torch.zeros_like(out)
    col = 0
    for t in range(T):
        lo, hi, bag = _bags(offsets, t, B)
        if hi > lo:
            rows = torch.from_numpy(np.asarray(indices[lo:hi], np.int64))
            W = torch.from_numpy(weights[t])
            x = W.index_select(0, rows).double()
            b = torch.from_numpy(bag)
            out[:, col:col + dims[t]].index_add_(0, b, x)
            aout[:, col:col + dims[t]].index_add_(0, b, x.abs())
        col += dims[t]
    return out.numpy(), aout.numpy()


def row_grads(B, dims, offsets, indices, grad, t):
    """(unique rows, g fp64 [U, D], g_abs fp64 [U, D]) of table t."""
    import torch

    lo, hi, bag = _bags(offsets, t, B)
    col = int(sum(dims[:t]))
    if hi == lo:
        return np.zeros(0, np.uint32), np.zeros((0, dims[t])), np.zeros((0, dims[t]))
    rows = np.asarray(indices[lo:hi], np.int64)
    uq, inv = np.unique(rows, return_inverse=True)
    gsrc = torch.from_numpy(np.ascontiguousarray(grad[:, col:col + dims[t]], np.float32)).double()
    g = torch.zeros(uq.size, dims[t], dtype=torch.float64)
    ga = torch.zeros_like(g)
    x = gsrc.index_select(0, torch.from_numpy(bag))
    ii = torch.from_numpy(inv.astype(np.int64))
    g.index_add_(0, ii, x)
    ga.index_add_(0, ii, x.abs())
    return uq.astype(np.uint32), g.numpy(), ga.numpy()


def update(w, m, g, ga, opt, lr, eps):
    """One row-wise update of rows w [U, D] (fp32 in), momentum m [U] (or None)
    with exact gradients g.  Returns (w_new fp64, m_new fp64 or None,
    w_bound, m_bound): the fp32 kernels must land within the bounds."""
    w = w.astype(np.float64)
    D = w.shape[1]
    if opt == "sgd":
        step = lr * g
        step_abs = lr * ga
        return w - step, None, RTOL * (np.abs(w - step) + step_abs) + 1e-30, None
    m0 = m.astype(np.float64)
    m1 = m0 + (g * g).sum(axis=1) / D
    m1_abs = m0 + (ga * ga).sum(axis=1) / D
    mult = lr / (np.sqrt(m1) + eps)
    step = mult[:, None] * g
    step_abs = mult[:, None] * ga
    return (w - step, m1, RTOL * (np.abs(w - step) + step_abs) + 1e-30,
            RTOL * m1_abs + 1e-30)


def check(got, want, bound, what):
    """Asserts |got - want| <= bound elementwise; returns the worst ratio."""
    got = np.asarray(got, np.float64)
    err = np.abs(got - want)
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} elements outside 1e-5 of the fp64 oracle; "
                             f"first at {tuple(i)}: got {got[tuple(i)]!r} want {want[tuple(i)]!r} "
                             f"bound {bound[tuple(i)]!r}")
    return float((err / bound).max()) if err.size else 0.0
