"""ctypes mirror of the C-ABI structs in include/mgcuda.h.

Plain data definitions shared by the product wrapper (_lib.py / api.py) and
the test-side oracle bindings (tests/oracle_bind.py).  Field order and types
must match include/mgcuda.h exactly; tests/test_abi.py checks the sizes.
"""
import ctypes as C

MG_OK, MG_EINVAL, MG_ELOGIC, MG_EDOMAIN, MG_ECUDA, MG_ENOMEM, MG_EUNSUPPORTED = range(7)
MG_F32, MG_F64 = 0, 1
MG_EXP_RATE, MG_MULT_NOISE, MG_MINI_RENDER = 0, 1, 2
MG_OPT_META, MG_OPT_ADAM = 0, 1
MG_TRAJ_OPTIMISE, MG_TRAJ_SCRIPTED_LINEAR, MG_TRAJ_SCRIPTED_EXP = 0, 1, 2
MG_DIFF_NORM_GLOBAL, MG_DIFF_NORM_PER_PARAM = 0, 1
MG_RNG_MT64, MG_RNG_PHILOX = 0, 1

PROBLEMS = {"exp-rate": MG_EXP_RATE, "mult-noise": MG_MULT_NOISE, "mini-render": MG_MINI_RENDER}
OPTIMIZERS = {"meta": MG_OPT_META, "adam": MG_OPT_ADAM}
TRAJECTORIES = {"optimise": MG_TRAJ_OPTIMISE, "scripted-linear": MG_TRAJ_SCRIPTED_LINEAR,
                "scripted-exp": MG_TRAJ_SCRIPTED_EXP}
DIFF_NORMS = {"global": MG_DIFF_NORM_GLOBAL, "per-param": MG_DIFF_NORM_PER_PARAM}


class ExperimentConfigC(C.Structure):
    """mg_experiment_config (include/mgcuda.h) == ExperimentConfig (harness.hpp:18-67)."""
    _fields_ = [
        ("problem", C.c_int32), ("optimizer", C.c_int32), ("iterations", C.c_int32),
        ("replicates", C.c_int32), ("seed", C.c_uint64),
        ("lr", C.c_double), ("beta_f", C.c_double), ("beta_delta", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps_step", C.c_double),
        ("eps_alpha", C.c_double), ("adam_eps", C.c_double),
        ("dim", C.c_int32), ("samples_per_iter", C.c_int32), ("sigma", C.c_double),
        ("target_mean", C.c_double), ("rate_init", C.c_double),
        ("pixel_count", C.c_int32), ("spp", C.c_int32), ("problem_seed", C.c_uint64),
        ("albedo_init", C.c_double), ("exponent_max", C.c_double),
        ("trajectory", C.c_int32), ("diff_norm", C.c_int32), ("traj_rate", C.c_double),
        ("no_alpha_clip", C.c_int32), ("independent_variance_samples", C.c_int32),
        ("non_zero_centred", C.c_int32), ("coord", C.c_int32),
        ("converge_threshold", C.c_double),
        ("dtype", C.c_int32), ("rng", C.c_int32),
    ]


class Moment2Scalars(C.Structure):
    _fields_ = [("decay", C.c_double), ("decay_pow", C.c_double), ("count", C.c_int64)]


class MetaParams(C.Structure):
    _fields_ = [("lr", C.c_double), ("eps_step", C.c_double), ("eps_alpha", C.c_double),
                ("clip_enabled", C.c_int32)]


class AdamScalars(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("beta1_pow", C.c_double), ("beta2_pow", C.c_double),
                ("t", C.c_int64)]


class UpdateScalars(C.Structure):
    _fields_ = [("ssn", C.c_double), ("changed", C.c_double), ("loss", C.c_double),
                ("nonfinite", C.c_double), ("diff_decay_pow", C.c_double),
                ("diff_count", C.c_int64), ("ssn_used", C.c_double), ("prop_decay_pow", C.c_double)]


class MetaUpdateArgs(C.Structure):
    _fields_ = [("meta", MetaParams), ("prop_coef", C.c_double), ("beta_delta", C.c_double),
                ("first_step", C.c_int32), ("diff_norm", C.c_int32), ("project", C.c_int32),
                ("ssn_from_host", C.c_int32), ("proj_lo", C.c_double), ("ssn_host", C.c_double),
                ("proj_hi", C.c_double), ("beta_f", C.c_double), ("prop_coef_device", C.c_int32),
                ("prop_pow_advance", C.c_int32)]


class MetaExtras(C.Structure):
    _fields_ = [("vprop", C.c_void_p), ("vdiff", C.c_void_p), ("params_prev", C.c_void_p),
                ("target", C.c_void_p), ("delta_out", C.c_void_p)]


class RenderArgs(C.Structure):
    _fields_ = [("update", MetaUpdateArgs), ("spp", C.c_int32), ("rng_kind", C.c_int32),
                ("key", C.c_uint64), ("iteration", C.c_uint32), ("stream", C.c_uint32),
                ("pixel_offset", C.c_uint32), ("record_plus1", C.c_int32)]


class RunRecordC(C.Structure):
    _fields_ = [("iterations_run", C.c_int32), ("status", C.c_int32),
                ("draws_used", C.c_int64), ("evals_used", C.c_int64)]


SERIES_NAMES = ("param_err", "loss", "prop", "diff", "grad_est", "est_var", "alpha", "delta",
                "true_grad", "step_sq_norm", "param")


class RunSeriesC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in SERIES_NAMES]


def fresh_scalars():
    """Initial mg_update_scalars of a run: no step taken, diff EMA empty."""
    return UpdateScalars(ssn=0.0, changed=0.0, loss=float("nan"), nonfinite=0.0,
                         diff_decay_pow=1.0, diff_count=0, ssn_used=0.0, prop_decay_pow=1.0)


def config_from(**kw):
    """ExperimentConfigC with the reference defaults (harness.hpp:18-67) and
    string-valued fields accepted the way the reference CLI spells them."""
    c = ExperimentConfigC()
    defaults = dict(problem="exp-rate", optimizer="meta", iterations=100, replicates=1, seed=0,
                    lr=0.01, beta_f=0.9, beta_delta=0.5, beta1=0.9, beta2=0.999, eps_step=1e-8,
                    eps_alpha=1e-30, adam_eps=1e-8, dim=4, sigma=1.0, samples_per_iter=32,
                    target_mean=2.0, rate_init=2.0, pixel_count=8, spp=4, problem_seed=1234,
                    albedo_init=0.1, exponent_max=4.0, trajectory="optimise", traj_rate=0.05,
                    no_alpha_clip=False, independent_variance_samples=False,
                    non_zero_centred=False, diff_norm="global", coord=0,
                    converge_threshold=-1.0, dtype=MG_F64, rng=MG_RNG_MT64)
    unknown = set(kw) - set(defaults) - {"threads", "out_csv", "out_json"}
    if unknown:
        raise TypeError(f"unknown config fields: {sorted(unknown)}")
    defaults.update({k: v for k, v in kw.items() if k in defaults})
    maps = {"problem": PROBLEMS, "optimizer": OPTIMIZERS, "trajectory": TRAJECTORIES,
            "diff_norm": DIFF_NORMS}
    for k, v in defaults.items():
        if k in maps and isinstance(v, str):
            if v not in maps[k]:
                raise ValueError(f"unknown {k} '{v}' (valid: {', '.join(maps[k])})")
            v = maps[k][v]
        if k == "dtype" and isinstance(v, str):
            v = {"f32": MG_F32, "f64": MG_F64}[v]
        if k == "rng" and isinstance(v, str):
            v = {"mt64": MG_RNG_MT64, "philox": MG_RNG_PHILOX}[v]
        setattr(c, k, int(v) if isinstance(v, bool) else v)
    return c


def config_text(**kw):
    """key=value;... text understood by oracle/ref/ref_capi.cpp parse_config."""
    parts = []
    for k, v in kw.items():
        if isinstance(v, bool):
            v = int(v)
        parts.append(f"{k}={v!r}" if isinstance(v, float) else f"{k}={v}")
    return ";".join(parts)
