"""CPU suite: pin the oracle (oracle/oracle.c) to the reference's known answers.

The oracle is the checker for every GPU parity test, so it is pinned first:
against the golden fixtures recorded from the unmodified reference library
(tools/make_golden.py) and, where the compiled reference is present, against
the reference itself on fresh seeded inputs.
"""
import math

import numpy as np
import pytest

from conftest import assert_stats_equal, golden_stats, golden_trace, load_golden

import oracle


def test_hash_value_goldens(coracle):
    # tests/test_workload.cpp:50-57
    assert coracle.hash_value(42, 1 << 32) == 3564271138
    assert coracle.hash_value(7, 1000) == 604
    for x in (0, 1, 42, 0xFFFFFFFFFFFFFFFF):
        assert coracle.hash_value(x, 1) == 0
    with pytest.raises(oracle.OracleError):
        coracle.hash_value(1, 0)
    for raw, H, want in load_golden("hash_value.json")["cases"]:
        assert coracle.hash_value(int(raw), int(H)) == int(want)


def _oracle_profile(coracle, tr, rate, seed, raw=None):
    return coracle.profile(tr.tables, tr.num_samples, tr.rec_sample, tr.rec_table, tr.rec_offset,
                           tr.rec_len, tr.ids, rate, seed, raw_ids=raw)


@pytest.mark.parametrize("name", list(load_golden("profile.json")))
def test_profile_matches_reference_goldens(coracle, name):
    case = load_golden("profile.json")[name]
    raw = case.get("raw_ids")
    tr = golden_trace(case["trace"], raw)
    got = _oracle_profile(coracle, tr, case["rate"], case["seed"], raw=tr.raw_ids)
    assert_stats_equal(got, golden_stats(case["stats"]))


def test_worked_example_values(coracle):
    # tests/test_profiler.cpp:53-62 (Fig. 3)
    case = load_golden("profile.json")["worked_example"]
    st = _oracle_profile(coracle, golden_trace(case["trace"]), 1.0, 0)
    assert st[0]["coverage"] == 1.0 and abs(st[0]["avg_pooling"] - 11 / 3) < 1e-12
    assert abs(st[1]["coverage"] - 1 / 3) < 1e-12 and st[1]["avg_pooling"] == 3.0
    assert st[0]["total_accesses"] == 11 and st[0]["distinct_rows_accessed"] == 6


def icdf_prefix_scan(counts):
    """tests/oracles.hpp:38-54 restated: literal scan with long-double-style need."""
    c = sorted((int(x) for x in counts), reverse=True)
    total = sum(c)
    out = [0] * 101
    for i in range(1, 101):
        # 100*cum >= i*total  <=>  cum >= total*i/100 (exact in integers)
        cum = k = 0
        while cum * 100 < i * total and k < len(c):
            cum += c[k]
            k += 1
        out[i] = k
    return out


def test_build_icdf_goldens_and_prefix_scan(coracle):
    for case in load_golden("build_icdf.json")["cases"]:
        got = coracle.build_icdf(case["counts"])
        assert list(got) == case["icdf"]
    # tests/test_profiler.cpp:103-119: 1000 random vectors vs the scan oracle
    rng = np.random.default_rng(2024)
    for _ in range(1000):
        n = int(rng.integers(1, 1000))
        c = rng.integers(0, 100, n)
        if c.sum() == 0:
            c[0] = 1
        assert list(coracle.build_icdf(c)) == icdf_prefix_scan(c)
    with pytest.raises(oracle.OracleError):
        coracle.build_icdf([0, 0, 0])


def test_build_icdf_shapes(coracle):
    # tests/test_profiler.cpp:83-101
    u = coracle.build_icdf([7] * 200)
    assert u[0] == 0 and u[50] == 100 and u[100] == 200
    t = coracle.build_icdf([90, 10])
    assert all(t[i] == 1 for i in range(1, 91)) and all(t[i] == 2 for i in range(91, 101))


def test_remap_goldens(coracle):
    for case in load_golden("remap.json")["cases"]:
        ent, slow = coracle.build_remap(case["hash_size"], case["hbm_rows"], case["rows_by_rank"],
                                        case["omit"])
        assert list(ent) == case["entries"]
        assert slow == case["slow_rows_allocated"]
    with pytest.raises(oracle.OracleError):
        coracle.build_remap(3, 4, [2, 0, 1])
    with pytest.raises(oracle.OracleError):
        coracle.build_remap(1 << 31, 0, [])


def report_from_counts(tables, plan, system, batches, hbm_t, tot_t):
    """core/src/simulator.cpp:96-137 applied to exact per-table counts."""
    gpu_of = dict(zip(plan["table_id"], plan["gpu"]))
    M = system["num_gpus"]
    hbm = [0] * M
    uvm = [0] * M
    hb = [0.0] * M
    ub = [0.0] * M
    for j, t in enumerate(tables):
        g = gpu_of[t.table_id]
        rb = float(t.dim * t.elem_bytes)
        hbm[g] += int(hbm_t[j])
        uvm[g] += int(tot_t[j] - hbm_t[j])
        hb[g] += float(hbm_t[j]) * rb
        ub[g] += float(tot_t[j] - hbm_t[j]) * rb
    bi = float(batches)
    cost = [(hb[g] / system["bw_hbm"] + ub[g] / system["bw_uvm"]) / bi for g in range(M)]
    total = sum(hbm) + sum(uvm)
    # plain left-to-right double sums (Python 3.12's sum() is compensated)
    s = 0.0
    for c in cost:
        s += c
    mean = s / M
    var = 0.0
    for c in cost:
        var += (c - mean) * (c - mean)
    return dict(hbm_accesses=[h / bi for h in hbm], uvm_accesses=[u / bi for u in uvm],
                est_iter_cost=cost, batches=batches, total_accesses=total,
                min_cost=min(cost), max_cost=max(cost), mean_cost=mean,
                stddev_cost=math.sqrt(var / M),
                uvm_access_fraction=(sum(uvm) / total) if total else 0.0,
                table_fast_fraction=[float(hbm_t[j]) / float(tot_t[j]) if tot_t[j] else math.nan
                                     for j in range(len(tables))])


def check_report(got, want):
    for k, w in want.items():
        g = got[k]
        if isinstance(w, str):
            w = float.fromhex(w)
        if isinstance(w, list):
            for a, b in zip(g, w):
                assert (math.isnan(a) and math.isnan(b)) or a == b, (k, a, b)
        else:
            assert g == w, (k, g, w)


def test_simulate_goldens(coracle):
    for case in load_golden("simulate.json")["cases"]:
        tr = golden_trace(case["trace"])
        plan = case["plan"]
        gpu_of = dict(zip(plan["table_id"], plan["gpu"]))
        rem = {r["table_id"]: np.array(r["entries"], np.int32) for r in case["remaps"]}
        B = case["batch_size"]
        batches = tr.num_samples // B
        hbm, uvm, tf, tt = coracle.simulate_counts(
            tr.tables, tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len, tr.ids,
            [gpu_of[t.table_id] for t in tr.tables], [rem[t.table_id] for t in tr.tables],
            case["system"]["num_gpus"], batches * B)
        check_report(report_from_counts(tr.tables, plan, case["system"], batches, tf, tt),
                     case["report"])


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_oracle_matches_reference_on_seeded_traces(coracle):
    R = oracle.Ref()
    S = oracle.Spec
    rng = np.random.default_rng(3)
    for trial in range(3):
        wl = []
        for j in range(int(rng.integers(1, 5))):
            H = int(rng.integers(1, 50000))
            wl.append((S(j * 3 + 1, int(rng.integers(1, 60000)), H, 4, 4),
                       (float(rng.uniform(0, 1.6)), float(rng.uniform(1, 12)),
                        float(rng.uniform(0.05, 1)), int(rng.integers(0, 3)))))
        tr = R.generate_trace(wl, int(rng.integers(100, 5000)), int(rng.integers(0, 1 << 40)))
        for rate, seed in [(1.0, 0), (float(rng.uniform(0.05, 1)), int(rng.integers(0, 99)))]:
            want = R.profile(tr, rate, seed)
            got = _oracle_profile(coracle, tr, rate, seed)
            assert_stats_equal(got, want)
        R.free_trace(tr)


def test_emb_forward_oracle_matches_torch(coracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    dims = [8, 16, 4]
    B = 33
    Ws = [coracle.init_table(7, t, 50 + t, d, 0.1) for t, d in enumerate(dims)]
    lens = rng.integers(0, 6, len(dims) * B)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    idx = np.concatenate([rng.integers(0, 50 + (i // B), l) for i, l in enumerate(lens)]).astype(np.uint32)
    out = coracle.emb_forward(B, dims, offsets, idx, Ws)
    col = 0
    for t, d in enumerate(dims):
        o = offsets[t * B:(t + 1) * B + 1].astype(np.int64)
        ref = torch.nn.functional.embedding_bag(
            torch.from_numpy(idx[o[0]:o[-1]].astype(np.int64)), torch.from_numpy(Ws[t]),
            torch.from_numpy(o[:-1] - o[0]), mode="sum")
        np.testing.assert_allclose(out[:, col:col + d], ref.numpy(), rtol=1e-6, atol=1e-7)
        col += d


def test_emb_backward_sgd_oracle_matches_autograd(coracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(6)
    dims = [8, 12]
    B = 40
    H = [30, 20]
    Ws = [coracle.init_table(3, t, H[t], d, 0.5) for t, d in enumerate(dims)]
    lens = rng.integers(0, 5, len(dims) * B)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    idx = np.concatenate([rng.integers(0, H[i // B], l) for i, l in enumerate(lens)]).astype(np.uint32)
    grad = rng.standard_normal((B, sum(dims))).astype(np.float32)
    ref = []
    col = 0
    for t, d in enumerate(dims):
        w = torch.tensor(Ws[t], requires_grad=True)
        o = offsets[t * B:(t + 1) * B + 1].astype(np.int64)
        y = torch.nn.functional.embedding_bag(torch.from_numpy(idx[o[0]:o[-1]].astype(np.int64)), w,
                                              torch.from_numpy(o[:-1] - o[0]), mode="sum")
        (y * torch.from_numpy(grad[:, col:col + d])).sum().backward()
        ref.append((w - 0.05 * w.grad).detach().numpy())
        col += d
    Wc = [w.copy() for w in Ws]
    coracle.emb_backward(B, dims, offsets, idx, grad, Wc, None, 0, 0.05, 1e-8)
    for a, b in zip(Wc, ref):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


# --------------------------------------------------------------- fp64 EmbeddingBag oracle
def test_emb64_forward_matches_torch_embedding_bag(coracle):
    """oracle/emb64.py (the independent fp64 oracle of the operator) against
    torch.nn.functional.embedding_bag(mode="sum") in float64."""
    torch = pytest.importorskip("torch")
    from oracle import emb64

    rng = np.random.default_rng(11)
    dims, H, B = [8, 64, 4], [300, 41, 7], 97
    Ws = [coracle.init_table(5, t, H[t], d, 0.3) for t, d in enumerate(dims)]
    lens = rng.integers(0, 9, len(dims) * B)
    lens[rng.random(lens.size) < 0.1] = 0
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    idx = np.concatenate([rng.integers(0, H[i // B], l) for i, l in enumerate(lens)]).astype(np.uint32)
    got, gabs = emb64.forward(B, dims, offsets, idx, Ws)
    col = 0
    for t, d in enumerate(dims):
        o = offsets[t * B:(t + 1) * B + 1].astype(np.int64)
        ref = torch.nn.functional.embedding_bag(
            torch.from_numpy(idx[o[0]:o[-1]].astype(np.int64)), torch.from_numpy(Ws[t]).double(),
            torch.from_numpy(o[:-1] - o[0]), mode="sum")
        np.testing.assert_allclose(got[:, col:col + d], ref.numpy(), rtol=1e-13, atol=1e-15)
        assert (gabs[:, col:col + d] >= np.abs(got[:, col:col + d]) - 1e-15).all()
        col += d
    # the C oracle's fp32 forward is inside the fp64 oracle's bound
    emb64.check(coracle.emb_forward(B, dims, offsets, idx, Ws), got, emb64.RTOL * gabs + 1e-30, "fwd")


@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_emb64_update_matches_autograd_and_adagrad_definition(coracle, opt):
    """fp64 row gradients = autograd of sum(pooled * grad) (float64); the
    row-wise update is FBGEMM's (exact row-wise Adagrad: one state per row,
    mean of squared gradient); the fp32 C oracle (the kernels' reduction
    tree) lands inside the fp64 bound."""
    torch = pytest.importorskip("torch")
    from oracle import emb64

    rng = np.random.default_rng(12)
    dims, H, B = [16, 8], [60, 25], 120
    lens = rng.integers(0, 7, len(dims) * B)
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    idx = np.concatenate([np.minimum(rng.zipf(1.3, l) - 1, H[i // B] - 1)
                          for i, l in enumerate(lens)]).astype(np.uint32)
    Ws = [coracle.init_table(8, t, H[t], d, 0.5) for t, d in enumerate(dims)]
    grad = rng.standard_normal((B, sum(dims))).astype(np.float32)
    lr, eps = 0.3, 1e-8
    mom = [np.full(h, 0.25, np.float32) for h in H]
    Wc, Mc = [w.copy() for w in Ws], [m.copy() for m in mom]
    coracle.emb_backward(B, dims, offsets, idx, grad, Wc, Mc if opt != "sgd" else None,
                         0 if opt == "sgd" else 1, lr, eps)
    col = 0
    for t, d in enumerate(dims):
        w = torch.tensor(Ws[t], dtype=torch.float64, requires_grad=True)
        o = offsets[t * B:(t + 1) * B + 1].astype(np.int64)
        y = torch.nn.functional.embedding_bag(torch.from_numpy(idx[o[0]:o[-1]].astype(np.int64)), w,
                                              torch.from_numpy(o[:-1] - o[0]), mode="sum")
        (y * torch.from_numpy(grad[:, col:col + d]).double()).sum().backward()
        rows, g, ga = emb64.row_grads(B, dims, offsets, idx, grad, t)
        np.testing.assert_allclose(g, w.grad.numpy()[rows], rtol=1e-13, atol=1e-14)
        wn, mn, wb, mb = emb64.update(Ws[t][rows], mom[t][rows], g, ga, opt, lr, eps)
        if opt == "sgd":
            np.testing.assert_allclose(wn, (w - lr * w.grad).detach().numpy()[rows], rtol=1e-13)
        else:
            gg = w.grad.numpy()[rows]
            m1 = mom[t][rows].astype(np.float64) + (gg * gg).mean(axis=1)
            np.testing.assert_allclose(mn, m1, rtol=1e-13)
            np.testing.assert_allclose(wn, Ws[t][rows] - lr * gg / (np.sqrt(m1) + eps)[:, None], rtol=1e-12)
            emb64.check(Mc[t][rows], mn, mb, "momentum")
        emb64.check(Wc[t][rows], wn, wb, "weights")
        col += d
