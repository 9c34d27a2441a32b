"""F2: across-replicate aggregation on the device
(csrc/aggregate.cu) against the reference's host reduction
(harness.cpp:274-302, stats.hpp:44-68) as restated by api.aggregate —
bit-identical, including ragged replicate lengths, empty columns, a single
replicate, NaN values and the maximum replicate count."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2309_15676_b200 import api
    return api


def _host_stats(series, runs):
    """stats.hpp on the host (api._column_stats, itself pinned by the
    byte-identical CSV tests)."""
    from paper_2309_15676_b200 import api
    S, R, T = series.shape
    out = np.empty((S, 5, T))
    active = np.array([int(np.sum(runs > i)) for i in range(T)])
    for s in range(S):
        for i in range(T):
            out[s, :, i] = api._column_stats(series[s, runs > i, i])
    return out, active


def _same(a, b):
    """Bit-identical, NaN payloads aside."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


@pytest.mark.parametrize("S,R,T", [(1, 1, 5), (3, 7, 40), (2, 100, 300), (1, 1000, 17),
                                   (1, 8192, 3)])
def test_device_aggregate_matches_host(api, S, R, T):
    rs = np.random.RandomState(R + T)
    series = rs.standard_normal((S, R, T)) * np.exp(rs.uniform(-5, 5, (S, R, T)))
    runs = rs.randint(0, T + 1, R).astype(np.int32)   # ragged, some replicates empty
    runs[0] = T
    for r in range(R):
        series[:, r, runs[r]:] = np.nan       # entries past iterations_run are never read
    st, act = api.aggregate_series_device(torch.tensor(series, device="cuda"),
                                          torch.tensor(runs, device="cuda"))
    want, want_act = _host_stats(series, runs)
    assert np.array_equal(act.cpu().numpy(), want_act)
    got = st.cpu().numpy()
    assert _same(got, want)


def test_device_aggregate_empty_columns_and_nans(api):
    S, R, T = 1, 9, 6
    rs = np.random.RandomState(3)
    series = rs.standard_normal((S, R, T))
    series[0, 2, 1] = np.nan
    series[0, 5, 1] = np.nan
    runs = np.array([3, 3, 2, 1, 3, 2, 0, 3, 1], dtype=np.int32)   # columns 3..5 empty
    st, act = api.aggregate_series_device(torch.tensor(series, device="cuda"),
                                          torch.tensor(runs, device="cuda"))
    want, want_act = _host_stats(series, runs)
    got = st.cpu().numpy()
    assert np.array_equal(act.cpu().numpy(), want_act)
    assert _same(got, want)
    # empty column: mean/quantiles NaN, variance 0 (stats.hpp:46,56,63)
    assert math.isnan(got[0, 0, 4]) and got[0, 1, 4] == 0.0 and math.isnan(got[0, 2, 4])
    # a NaN in the sample poisons the mean like the reference's sequential sum
    assert math.isnan(got[0, 0, 1])


def test_device_aggregate_rejects_bad_arguments(api):
    with pytest.raises(api.InvalidArgument):
        api.aggregate_series_device(torch.zeros((1, 2, 3), device="cuda"),   # fp32 series
                                    torch.zeros(2, dtype=torch.int32, device="cuda"))
    with pytest.raises(api.InvalidArgument):
        api.aggregate_series_device(torch.zeros((1, 2, 3), dtype=torch.float64, device="cuda"),
                                    torch.zeros(3, dtype=torch.int32, device="cuda"))
    from paper_2309_15676_b200._lib import MgError
    with pytest.raises(MgError):
        api.aggregate_series_device(torch.zeros((1, 8193, 1), dtype=torch.float64, device="cuda"),
                                    torch.ones(8193, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("kw", [
    dict(problem="exp-rate", iterations=60, replicates=40, seed=11),
    dict(problem="mini-render", pixel_count=16, spp=8, iterations=50, replicates=12, seed=2),
    dict(problem="mult-noise", dim=4, iterations=80, replicates=30, seed=3, optimizer="adam",
         lr=0.05),
])
def test_run_experiment_device_aggregate_equals_host_aggregate(api, kw):
    """Same device run reduced on the device and on the host: identical
    statistics (bit for bit) and records."""
    cfg = api.ExperimentConfig(**kw)
    host = api.run_experiment(cfg)
    dev = api.run_experiment(cfg, device_aggregate=True)
    assert host.series_names == dev.series_names
    assert np.array_equal(host.active_replicates, dev.active_replicates)
    assert host.diverged_count == dev.diverged_count
    for a, b in zip(host.records, dev.records):
        assert (a.status, a.iterations_run, a.draws_used, a.evals_used) == \
            (b.status, b.iterations_run, b.draws_used, b.evals_used)
    for n in host.series_names:
        for f in ("mean", "variance", "median", "q25", "q75"):
            assert _same(getattr(host.stats[n], f), getattr(dev.stats[n], f)), (n, f)
