import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_trace(tj, raw_ids=None):
    from paper_2201_10095_b200.types import TableSpec, Trace

    tables = [TableSpec(**t) for t in tj["tables"]]
    raw = None if raw_ids is None else np.array([int(x) for x in raw_ids], np.uint64)
    return Trace(tables, tj["num_samples"], np.array(tj["rec_sample"], np.uint64),
                 np.array(tj["rec_table"], np.uint32), np.array(tj["rec_offset"], np.uint64),
                 np.array(tj["rec_len"], np.uint32),
                 ids=None if raw is not None else np.array(tj["ids"], np.uint32), raw_ids=raw)


def golden_stats(sj):
    return [dict(table_id=s["table_id"], coverage=float.fromhex(s["coverage"]),
                 avg_pooling=float.fromhex(s["avg_pooling"]),
                 distinct_rows_accessed=s["distinct_rows_accessed"],
                 total_accesses=s["total_accesses"],
                 icdf_steps=np.array(s["icdf_steps"], np.uint64),
                 access_cdf=np.array([float.fromhex(x) for x in s["access_cdf"]], np.float64),
                 rows_by_rank=np.array(s["rows_by_rank"], np.uint32)) for s in sj]


def assert_stats_equal(got, want):
    """Bit-exact FeatureStats comparison (got: FeatureStats or dict)."""
    assert len(got) == len(want)
    for g, w in zip(got, want):
        gd = g if isinstance(g, dict) else vars(g)
        for k in ("table_id", "distinct_rows_accessed", "total_accesses"):
            assert int(gd[k]) == int(w[k]), (k, gd[k], w[k])
        for k in ("coverage", "avg_pooling"):
            assert float(gd[k]) == float(w[k]), (k, gd[k], w[k])  # bit-exact doubles
        for k in ("icdf_steps", "access_cdf", "rows_by_rank"):
            a, b = np.asarray(gd[k]), np.asarray(w[k])
            assert a.shape == b.shape, (k, a.shape, b.shape)
            assert np.array_equal(a.view(np.uint64) if a.dtype == np.float64 else a,
                                  b.view(np.uint64) if b.dtype == np.float64 else b), k


@pytest.fixture(scope="session")
def cuda_ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_10095_b200 import default_context

    return default_context(0)


@pytest.fixture(scope="session")
def coracle():
    import oracle

    return oracle.C()
