"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE.  Run here (where /root/reference exists and
`make -C oracle/ref` has built oracle/_ref/libmetagrad_ref.so):

    python oracle/gen_golden.py

Every fixture is produced by calling the reference's own public API through
oracle/ref/ref_capi.cpp; the inputs (seeds, parameter vectors) are listed
below so the fixtures are reproducible.  The fixtures pin the C restatement
(oracle/metagrad_oracle.c) in tests/test_oracle_golden.py and are the
golden vectors the GPU parity tests compare against.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import RefLib  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    g = {}

    # 1. RNG streams (rng.hpp:23-36): first 2000 raw/uniform outputs of
    #    Rng::stream(s, r), plus a checksum (xor + sum mod 2^64) of 100000.
    for s in (0, 7, 42):
        for r in (0, 1, 999):
            raw = ref.rng_draws(s, r, 1, 100000)
            g[f"rng_raw_s{s}_r{r}"] = raw[:2000]
            g[f"rng_xor_s{s}_r{r}"] = np.bitwise_xor.reduce(raw)
            g[f"rng_sum_s{s}_r{r}"] = np.sum(raw, dtype=np.uint64)
            g[f"rng_uni_s{s}_r{r}"] = ref.rng_draws(s, r, 2, 2000)
            g[f"rng_upos_s{s}_r{r}"] = ref.rng_draws(s, r, 3, 2000)
    g["rng_engine_raw_seed5489"] = ref.rng_draws(5489, 0, 0, 10000)  # std 10000th-output check
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **g)

    # 2. Mini-render construction (problems.cpp:162-173) and sample pairs.
    g = {}
    for P, seed in ((16, 2024), (4096, 1), (8, 1234), (6, 11)):
        b, T, init = ref.minirender_gen(P, 4, seed)
        g[f"gen_P{P}_s{seed}_b"], g[f"gen_P{P}_s{seed}_T"] = b, T
    rs = np.random.RandomState(0)
    for P, spp, seed in ((16, 4, 2024), (4096, 2, 1), (6, 3, 11)):
        u = rs.random_sample(P * spp)
        u[0] = 0.0  # edge: pow(0, b)
        cross, mb = ref.minirender_kernel_terms(P, spp, seed, u)
        g[f"kt_P{P}_spp{spp}_u"], g[f"kt_P{P}_spp{spp}_cross"] = u, cross
        g[f"kt_P{P}_spp{spp}_mb"] = mb
        now = 0.1 + rs.random_sample(P)
        prev = now - 0.01 * rs.random_sample(P)
        g[f"sp_P{P}_spp{spp}_now"], g[f"sp_P{P}_spp{spp}_prev"] = now, prev
        for skip in (0, 2):
            prop, diff, ssn = ref.minirender_sample_pair(P, spp, seed, now, prev, 909, 3, skip)
            g[f"sp_P{P}_spp{spp}_k{skip}_prop"] = prop
            g[f"sp_P{P}_spp{spp}_k{skip}_diff"] = diff
            g[f"sp_P{P}_spp{spp}_k{skip}_ssn"] = np.float64(ssn)
        prop, diff, ssn = ref.minirender_sample_pair(P, spp, seed, now, now, 909, 3, 0)
        g[f"sp_P{P}_spp{spp}_same_prop"], g[f"sp_P{P}_spp{spp}_same_diff"] = prop, diff
    # exp-rate (problems.cpp:54-76) and mult-noise (:121-139)
    er = []
    for now, prev in ((2.0, 2.0), (1.25, 1.3), (0.8, 0.9), (0.5, 0.5)):
        for skip in (0, 1, 5):
            p, d, s, rc = ref.exprate_sample_pair(2.0, 32, now, prev, 808, 7, skip)
            er.append((now, prev, skip, p, d, s))
    g["exprate"] = np.array(er)
    p, d, s, rc = ref.exprate_sample_pair(2.0, 32, -0.5, 1.0, 1, 0, 0)
    g["exprate_domain_rc"] = np.int64(rc)
    target = np.zeros(4)
    now = np.array([1.5, -0.7, 2.2, 0.3])
    prev = np.array([1.45, -0.75, 2.14, 0.33])
    for skip in (0, 3):
        prop, diff, ssn = ref.multnoise_sample_pair(1.0, 2, target, now, prev, 404, 0, skip)
        g[f"mn_k{skip}_prop"], g[f"mn_k{skip}_diff"], g[f"mn_k{skip}_ssn"] = prop, diff, ssn
    np.savez_compressed(os.path.join(OUT, "problems.npz"), **g)

    # 3. Estimators: Moment2 runs, MetaEstimator steps from injected states,
    #    Adam runs (moment2.hpp:30-39, meta.hpp:90-113, adam.hpp:23-37).
    g = {}
    xs = rs.uniform(-2, 2, size=(50, 7))
    xs[3, 2] = 0.0
    for decay in (0.5, 0.9, 0.99):
        g[f"m2_d{decay}_xs"] = xs
        g[f"m2_d{decay}_out"] = ref.moment2_run(decay, xs)
    n = 257
    for k, clip in ((0, 1), (1, 1), (2, 0)):
        st = None if k == 0 else {"mean": rs.normal(size=n), "var": rs.uniform(0, 2, n),
                                  "alpha_prev": rs.uniform(-0.5, 0.99, n)}
        prop, diff = rs.normal(size=n), rs.normal(size=n) * 0.1
        vp, vd = rs.uniform(0, 3, n), rs.uniform(0, 0.5, n)
        if k == 0:
            diff = np.zeros(n)
            vd = np.zeros(n)
        out, delta, rc = ref.meta_step(0.01, 1e-8, 1e-30, clip, st, prop, diff, 0.02, vp, vd)
        g[f"meta{k}_in"] = np.stack([prop, diff, vp, vd])
        if st is not None:
            g[f"meta{k}_state_in"] = np.stack([st["mean"], st["var"], st["alpha_prev"]])
        g[f"meta{k}_state_out"] = np.stack([out["mean"], out["var"], out["alpha_prev"]])
        g[f"meta{k}_delta"] = delta
        g[f"meta{k}_clip"] = np.int64(clip)
    grads = rs.uniform(-3, 3, size=(40, 33))
    m, v, d = ref.adam_run(grads, lr=0.02)
    g["adam_grads"], g["adam_m"], g["adam_v"], g["adam_delta"] = grads, m, v, d
    np.savez_compressed(os.path.join(OUT, "estimators.npz"), **g)

    # 4. Full run_single records (harness.cpp:90-200) for the configurations
    #    the reference's own harness/acceptance tests exercise.
    g = {}
    runs = {
        "accept9": dict(problem="mini-render", pixel_count=16, spp=4, problem_seed=2024,
                        albedo_init=0.1, iterations=120, seed=909, lr=0.01),
        "accept9_noclip": dict(problem="mini-render", pixel_count=16, spp=4, problem_seed=2024,
                               iterations=120, seed=909, lr=0.01, no_alpha_clip=True),
        "noiseless": dict(problem="mult-noise", dim=1, sigma=0.0, samples_per_iter=1,
                          trajectory="scripted-linear", iterations=3),
        "scripted_exp": dict(problem="mult-noise", dim=1, sigma=1.0, samples_per_iter=4,
                             trajectory="scripted-exp", traj_rate=0.05, iterations=60, seed=606),
        "exprate": dict(problem="exp-rate", iterations=200, seed=808, lr=0.003, beta_f=0.99),
        "exprate_adam": dict(problem="exp-rate", optimizer="adam", iterations=100, seed=808,
                             lr=0.03),
        "multnoise_indep": dict(problem="mult-noise", dim=3, iterations=50, seed=5,
                                independent_variance_samples=True),
        "multnoise_perparam": dict(problem="mult-noise", dim=3, iterations=50, seed=6,
                                   diff_norm="per-param"),
        "diverge": dict(problem="mult-noise", dim=2, lr=1e300, iterations=10),
        "minirender_adam": dict(problem="mini-render", pixel_count=8, spp=3, optimizer="adam",
                                iterations=40, seed=77, lr=0.05),
        "s1_standin": dict(problem="mini-render", pixel_count=4096, spp=2, iterations=4,
                           seed=0, problem_seed=1, lr=0.01),
    }
    for name, kw in runs.items():
        for rep in ((0, 3) if name == "accept9" else (0,)):
            rec = ref.run_single(kw, rep)
            key = f"{name}_r{rep}"
            for k, v in rec.items():
                g[f"{key}__{k}"] = np.asarray(v)
            g[f"{key}__cfg"] = np.array(repr(kw))
    np.savez_compressed(os.path.join(OUT, "runs.npz"), **g)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
