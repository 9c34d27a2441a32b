"""F3: the reference's writers restated on the host — format_double
against the reference's own std::to_chars, json_double against its
nlohmann::json dump (oracle/_ref), and whole aggregate CSVs, summary JSONs
and per-replicate CSVs byte-identical for runs whose trajectories are
bit-exact."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from paper_2309_15676_b200 import report

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ref_fmt():
    from oracle_bind import REF_SO, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(REF_SO)
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]

    def f(v):
        buf = C.create_string_buffer(64)
        assert L.ref_format_double(v, buf, 64) == 0
        return buf.value.decode()
    return f


REF_EXE = os.path.join(ROOT, "oracle", "_ref", "run_experiment")


def ref_outputs_golden(kw, csv, js, rep_csv=None, rep=0):
    """The reference's run_experiment + all three writers (harness.cpp:305-427)."""
    import subprocess
    from paper_2309_15676_b200 import _abi
    if not os.path.exists(REF_EXE):
        pytest.skip("oracle/_ref not built")
    args = [REF_EXE, _abi.config_text(**kw), csv, js]
    if rep_csv:
        args += [rep_csv, str(rep)]
    subprocess.run(args, check=True, capture_output=True)


def ref_csv_golden(kw, path):
    """The reference's own run_experiment + CSV writer, in a separate process
    (its iostreams crash when numpy's bundled runtime shares the process)."""
    import subprocess
    from paper_2309_15676_b200 import _abi
    if not os.path.exists(REF_EXE):
        pytest.skip("oracle/_ref not built")
    subprocess.run([REF_EXE, _abi.config_text(**kw), path], check=True, capture_output=True)


def test_format_double_matches_std_to_chars():
    f = ref_fmt()
    rs = np.random.RandomState(0)
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 1e-5, 1e-4, 123456.0, 1e15, 1e16, 1e21, 1e22, 1e23,
            2.5e-300, 5e-324, 1.7976931348623157e308, float("inf"), float("-inf"), 0.5, 100.0,
            1234567.0, 0.001, 12.5, 1e100, 3.0e-7, 65536.0, 2.0 ** 53, 2.0 ** 60]
    vals += list(rs.standard_normal(3000))
    vals += list(np.exp(rs.uniform(-700, 700, 3000)))
    vals += [struct.unpack("<d", struct.pack("<Q", int(x)))[0]
             for x in rs.randint(0, 2 ** 62, 3000, dtype=np.int64)]
    vals += [float(k) for k in range(-50, 50)] + [k / 8 for k in range(-100, 100)]
    bad = [(v, report.format_double(v), f(v)) for v in vals
           if not np.isnan(v) and report.format_double(v) != f(v)]
    assert not bad, bad[:10]


def test_json_double_matches_nlohmann_dump():
    from oracle_bind import REF_SO, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    L = C.CDLL(REF_SO)
    L.ref_json_double.argtypes = [C.c_double, C.c_char_p, C.c_int]

    def ref(v):
        buf = C.create_string_buffer(64)
        assert L.ref_json_double(v, buf, 64) == 0
        return buf.value.decode()
    rs = np.random.RandomState(1)
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 0.01, 1e-3, 1e-4, 1e-5, 1.5e-5, 1e-30, 1e-8, 123456.0,
            1e14, 1e15, 1e16, 1.5e16, 1e21, 1e100, 5e-324, 1.7976931348623157e308, 0.5, 2.0 ** 53,
            float("nan"), float("inf"), float("-inf"), 100.0, 12.5, -0.000747712423299419]
    vals += list(rs.standard_normal(3000))
    vals += list(np.exp(rs.uniform(-700, 700, 3000)))
    vals += [struct.unpack("<d", struct.pack("<Q", int(x)))[0]
             for x in rs.randint(0, 2 ** 62, 20000, dtype=np.int64)]
    vals += [float(k) for k in range(-50, 50)] + [k / 8 for k in range(-100, 100)]
    vals += [2.0 ** k for k in range(-1074, 1024, 7)]          # lower-boundary-closer cases
    bad = [(v, report.json_double(v), ref(v)) for v in vals if report.json_double(v) != ref(v)]
    assert not bad, bad[:10]


@pytest.mark.parametrize("kw", [
    dict(problem="mult-noise", dim=2, iterations=25, replicates=6, seed=5),
    dict(problem="mult-noise", dim=3, iterations=30, replicates=5, seed=8, optimizer="adam",
         lr=0.05, converge_threshold=2.5),
])
def test_summary_json_bytes_match_reference_oracle(tmp_path, kw):
    """summary_json (harness.cpp:367-427) of oracle records == the
    reference's, byte for byte."""
    from test_dist_gloo import _oracle_run_fn
    from paper_2309_15676_b200.api import ExperimentConfig, aggregate
    ref_csv, ref_js = str(tmp_path / "ref.csv"), str(tmp_path / "ref.json")
    ref_outputs_golden(dict(kw, threads=1), ref_csv, ref_js)
    cfg = ExperimentConfig(**kw)
    rep = aggregate(cfg, _oracle_run_fn(cfg, 0, cfg.replicates))
    assert report.summary_json(rep).encode() == open(ref_js, "rb").read()


def test_csv_bytes_match_reference_oracle(tmp_path):
    """Aggregate CSV of oracle records (bit-exact with the reference for
    mult-noise) written by report.write_aggregate_csv == the reference's own
    writer, byte for byte."""
    from test_dist_gloo import _oracle_run_fn
    from paper_2309_15676_b200 import _abi
    from paper_2309_15676_b200.api import ExperimentConfig, aggregate
    kw = dict(problem="mult-noise", dim=2, iterations=25, replicates=6, seed=5)
    ref_csv = str(tmp_path / "ref.csv")
    ref_csv_golden(dict(kw, threads=1), ref_csv)
    cfg = ExperimentConfig(**kw)
    rep = aggregate(cfg, _oracle_run_fn(cfg, 0, 6))
    ours = str(tmp_path / "ours.csv")
    report.write_aggregate_csv(rep, ours)
    assert open(ours, "rb").read() == open(ref_csv, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [
    dict(problem="mult-noise", dim=2, iterations=25, replicates=6, seed=5),
    dict(problem="mult-noise", dim=1, sigma=1.0, samples_per_iter=4, trajectory="scripted-exp",
         traj_rate=0.05, iterations=40, replicates=50, seed=606),
    dict(problem="mult-noise", dim=3, iterations=30, replicates=9, seed=8, optimizer="adam",
         lr=0.05),
])
@pytest.mark.parametrize("device_aggregate", [False, True])
def test_device_run_csv_is_byte_identical_to_reference(tmp_path, kw, device_aggregate):
    """End to end: the device runner's report, written in the reference's
    format, equals the reference harness's CSV byte for byte (problems whose
    arithmetic has no transcendental functions are bit-exact on the device)."""
    from paper_2309_15676_b200 import api
    ref_csv = str(tmp_path / "ref.csv")
    ref_csv_golden(dict(kw, threads=1), ref_csv)
    rep = api.run_experiment(api.ExperimentConfig(**kw), device_aggregate=device_aggregate)
    ours = str(tmp_path / "ours.csv")
    report.write_aggregate_csv(rep, ours)
    assert open(ours, "rb").read() == open(ref_csv, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("kw,rep", [
    (dict(problem="mult-noise", dim=2, iterations=25, replicates=6, seed=5), 0),
    (dict(problem="mult-noise", dim=3, iterations=30, replicates=4, seed=8, optimizer="adam",
          lr=0.05), 2),
    (dict(problem="mult-noise", dim=1, sigma=1.0, samples_per_iter=4, trajectory="scripted-exp",
          traj_rate=0.05, iterations=40, replicates=3, seed=606, converge_threshold=1.9), 1),
    (dict(problem="mult-noise", dim=2, iterations=20, replicates=2, seed=9,
          diff_norm="per-param"), 1),
])
def test_device_run_all_writers_byte_identical_to_reference(tmp_path, kw, rep):
    """Device run -> the reference's three outputs: aggregate CSV, summary
    JSON (host- and device-aggregated) and the wide per-replicate CSV from
    the full device-recorded vectors — each byte-identical."""
    from paper_2309_15676_b200 import api
    ref_csv, ref_js, ref_rep = (str(tmp_path / n) for n in ("r.csv", "r.json", "rep.csv"))
    ref_outputs_golden(dict(kw, threads=1), ref_csv, ref_js, ref_rep, rep)
    cfg = api.ExperimentConfig(**kw)
    for dev_agg in (False, True):
        agg = api.run_experiment(cfg, device_aggregate=dev_agg)
        assert report.summary_json(agg).encode() == open(ref_js, "rb").read()
        ours = str(tmp_path / "ours.csv")
        report.write_aggregate_csv(agg, ours)
        assert open(ours, "rb").read() == open(ref_csv, "rb").read()
    rec = api.run_single(cfg, rep, full=True)
    ours_rep = str(tmp_path / "ours_rep.csv")
    report.write_replicate_csv(rec, ours_rep)
    assert open(ours_rep, "rb").read() == open(ref_rep, "rb").read()


def test_vectorised_aggregate_equals_per_column_stats():
    """harness.aggregate reduces every iteration column at once; it must
    equal _column_stats (stats.hpp:45-68) column by column, bit for bit,
    with ragged replicates (diverged early), NaN values, signed zeros,
    one-replicate and empty columns."""
    from paper_2309_15676_b200 import harness as H
    rs = np.random.RandomState(3)
    for R, T in ((1, 7), (2, 5), (9, 40), (33, 17)):
        cols = rs.standard_normal((R, T)) * 10 ** rs.uniform(-3, 3, (R, T))
        cols[rs.uniform(size=(R, T)) < 0.05] = np.nan
        cols[rs.uniform(size=(R, T)) < 0.05] = -0.0
        cols[:, 0] = -0.0
        runs = rs.randint(0, T + 1, R)
        runs[0] = T
        mask = runs[:, None] > np.arange(T)[None, :]
        got = H._stats_columns(cols, mask)
        for i in range(T):
            ref = H._column_stats(cols[mask[:, i], i])
            for k in range(5):
                a, b = np.float64(got[k][i]), np.float64(ref[k])
                assert (np.isnan(a) and np.isnan(b)) or a.tobytes() == b.tobytes(), (R, T, i, k, a, b)
