"""Reference-format reports of a device run:
byte-for-byte the outputs the reference harness writes (harness.cpp:305-427:
the aggregate CSV, the per-replicate wide CSV and the summary JSON), so a
user of the reference can diff outputs directly.

format_double restates std::to_chars(double) (harness.cpp:305-309): the
shortest digit string that round-trips, printed in fixed or scientific
(printf %e style, >= 2 exponent digits) notation, whichever is shorter,
fixed on a tie.
"""
from __future__ import annotations

import io
import math
from typing import IO, Union


def _shortest_digits(v: float):
    """(sign, digits, exp10) with v = 0.d1d2...dn * 10**exp10, shortest
    round-trip digits (Python's repr is shortest round-trip too)."""
    r = repr(abs(float(v)))
    mant, _, e = r.partition("e")
    exp = int(e) if e else 0
    ip, _, fp = mant.partition(".")
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    lead_zeros = len(ip + fp) - len((ip + fp).lstrip("0"))
    # position of the decimal point relative to the start of ip+fp is len(ip)
    point = len(ip) + exp - lead_zeros
    digits = digits.rstrip("0") or "0"
    return ("-" if math.copysign(1.0, v) < 0 else ""), digits, point


def format_double(v: float) -> str:
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign, d, point = _shortest_digits(v)
    n = len(d)
    # fixed
    if point <= 0:
        fixed = "0." + "0" * (-point) + d
    elif point >= n:
        # integral value: printf-style fixed notation prints the exact
        # integer (libstdc++ to_chars does the same), same length as d+zeros
        fixed = str(int(abs(v)))
    else:
        fixed = d[:point] + "." + d[point:]
    # scientific: d1.d2..dn e(point-1)
    e = point - 1
    sci = d[0] + ("." + d[1:] if n > 1 else "") + "e" + ("-" if e < 0 else "+") + \
        f"{abs(e):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def write_aggregate_csv(report, out: Union[str, IO[str]], tag: str = "",
                        with_header: bool = True) -> None:
    """harness.cpp:311-342."""
    buf = io.StringIO()
    if with_header:
        buf.write("iteration,statistic,value\n" if not tag else
                  "optimizer,iteration,statistic,value\n")
    prefix = f"{tag}," if tag else ""
    fields = (("mean", "mean"), ("var", "variance"), ("median", "median"), ("q25", "q25"),
              ("q75", "q75"))
    for i in range(report.config.iterations):
        for name in report.series_names:
            st = report.stats[name]
            for suffix, attr in fields:
                buf.write(f"{prefix}{i},{name}_{suffix},"
                          f"{format_double(float(getattr(st, attr)[i]))}\n")
        buf.write(f"{prefix}{i},active_replicates,{int(report.active_replicates[i])}\n")
    text = buf.getvalue()
    if isinstance(out, str):
        with open(out, "w", newline="") as f:
            f.write(text)
    else:
        out.write(text)


# ---- nlohmann::json's double -> text (Grisu2, Loitsch 2010, as restated in
# nlohmann/json detail::dtoa_impl).  Grisu2 is NOT always shortest (about
# 0.03% of doubles get one more digit than std::to_chars), so summary_json
# needs this exact digit generator to be byte-identical.
_M64 = (1 << 64) - 1


def _cached_pow10(k: int):
    """(f, e) with f * 2**e ~= 10**k, f a rounded 64-bit normalised significand."""
    from fractions import Fraction
    v = Fraction(10) ** k
    e = v.numerator.bit_length() - v.denominator.bit_length() - 64
    while True:
        f = v / Fraction(2) ** e
        if f < 2 ** 63:
            e -= 1
        elif f >= 2 ** 64:
            e += 1
        else:
            break
    fi = int(f)
    if f - fi >= Fraction(1, 2):
        fi += 1
    return fi, e


_CACHED = None


def _cached_for_binary_exponent(e: int):
    global _CACHED
    if _CACHED is None:
        _CACHED = [(_cached_pow10(k), k) for k in range(-300, 325, 8)]
    f = -60 - e - 1                                    # kAlpha - e - 1
    k = int(f * 78913 / (1 << 18)) if f * 78913 >= 0 else -((-f * 78913) // (1 << 18))
    k += 1 if f > 0 else 0
    index = (300 + k + 7) // 8
    (cf, ce), ck = _CACHED[index]
    return cf, ce, ck


def _diy_mul(xf, xe, yf, ye):
    return ((xf * yf + (1 << 63)) >> 64) & _M64, xe + ye + 64


def _diy_normalize(f, e):
    shift = 64 - f.bit_length()
    return (f << shift) & _M64, e - shift


def _grisu2_digits(v: float):
    """(digits, decimal_exponent) with |v| ~= int(digits) * 10**decimal_exponent."""
    import struct
    bits = struct.unpack("<Q", struct.pack("<d", abs(v)))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    if E == 0:
        vf, ve = F, 1 - 1075
    else:
        vf, ve = F + (1 << 52), E - 1075
    lower_closer = F == 0 and E > 1
    mpf, mpe = 2 * vf + 1, ve - 1
    if lower_closer:
        mmf, mme = 4 * vf - 1, ve - 2
    else:
        mmf, mme = 2 * vf - 1, ve - 1
    wpf, wpe = _diy_normalize(mpf, mpe)
    wmf, wme = mmf << (mme - wpe), wpe                  # normalize_to(m-, w+.e)
    wf, we = _diy_normalize(vf, ve)
    cf, ce, ck = _cached_for_binary_exponent(wpe)
    w_f, w_e = _diy_mul(wf, we, cf, ce)
    lo_f, _ = _diy_mul(wmf, wme, cf, ce)
    hi_f, hi_e = _diy_mul(wpf, wpe, cf, ce)
    Mm, Mp = lo_f + 1, hi_f - 1
    dec = -ck
    # grisu2_digit_gen
    delta = Mp - Mm
    dist = Mp - w_f
    sh = -hi_e
    one = 1 << sh
    p1, p2 = Mp >> sh, Mp & (one - 1)
    digits = []
    pow10, k = 1, 1
    for kk, pw in ((10, 10 ** 9), (9, 10 ** 8), (8, 10 ** 7), (7, 10 ** 6), (6, 10 ** 5),
                   (5, 10 ** 4), (4, 1000), (3, 100), (2, 10)):
        if p1 >= pw:
            pow10, k = pw, kk
            break
    n = k
    while n > 0:
        d, p1 = divmod(p1, pow10)
        digits.append(d)
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            dec += n
            return _grisu2_round(digits, dist, delta, rest, pow10 << sh), dec
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        d, p2 = p2 >> sh, p2 & (one - 1)
        digits.append(d)
        m += 1
        delta *= 10
        dist *= 10
        if p2 <= delta:
            break
    dec -= m
    return _grisu2_round(digits, dist, delta, p2, one), dec


def _grisu2_round(digits, dist, delta, rest, ten_k):
    while rest < dist and delta - rest >= ten_k and \
            (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
        digits[-1] -= 1
        rest += ten_k
    return "".join(str(d) for d in digits)


def json_double(v: float) -> str:
    """A double as nlohmann::json's dump prints it (the reference's
    summary_json, harness.cpp:367-427): Grisu2 digits; fixed notation with
    at least one fractional digit when the decimal point position n lies in
    (-4, 15], otherwise d[.ddd]e±XX; NaN/inf as null."""
    v = float(v)
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    d, dec = _grisu2_digits(v)
    k = len(d)
    n = k + dec
    if k <= n <= 15:
        body = d + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        body = d[:n] + "." + d[n:]
    elif -4 < n <= 0:
        body = "0." + "0" * (-n) + d
    else:
        e = n - 1
        body = (d if k == 1 else d[0] + "." + d[1:]) + "e" + ("-" if e < 0 else "+") + \
            (f"{abs(e):02d}")
    return sign + body


def _json_string(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch in "\b\f\n\r\t":
            out.append({"\b": "\\b", "\f": "\\f", "\n": "\\n", "\r": "\\r", "\t": "\\t"}[ch])
        elif o < 0x20:
            out.append(f"\\u{o:04x}")
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _json_dump(obj, indent: int = 2, level: int = 0) -> str:
    """nlohmann::ordered_json::dump(2) for dicts of str/int/float."""
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        pad = " " * (indent * (level + 1))
        items = [f"{pad}{_json_string(k)}: {_json_dump(v, indent, level + 1)}"
                 for k, v in obj.items()]
        return "{\n" + ",\n".join(items) + "\n" + " " * (indent * level) + "}"
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return json_double(obj)
    if isinstance(obj, str):
        return _json_string(obj)
    raise TypeError(f"unsupported JSON value {obj!r}")


def summary_json(report) -> str:
    """harness.cpp:367-427: schema_version, config echo, final-iteration
    statistics, convergence iteration, divergence count, per-iteration draw
    and evaluation counts — byte-identical to the reference's output."""
    cfg = report.config
    j = {"schema_version": 1, "problem": cfg.problem, "optimizer": cfg.optimizer,
         "iterations": int(cfg.iterations), "replicates": int(cfg.replicates),
         "seed": int(cfg.seed), "lr": float(cfg.lr), "beta_f": float(cfg.beta_f),
         "beta_delta": float(cfg.beta_delta), "trajectory": cfg.trajectory,
         "diverged_replicates": int(report.diverged_count)}
    last = cfg.iterations - 1
    finals = {}
    for name in report.series_names:
        st = report.stats[name]
        finals[name] = {"mean": float(st.mean[last]), "median": float(st.median[last]),
                        "q25": float(st.q25[last]), "q75": float(st.q75[last])}
    j["final"] = finals
    conv = -1
    if cfg.converge_threshold > 0.0 and "param_err" in report.stats:
        med = report.stats["param_err"].median
        for i in range(cfg.iterations):
            if med[i] < cfg.converge_threshold:
                conv = i
                break
    j["convergence_iteration"] = conv
    j["converge_threshold"] = float(cfg.converge_threshold)
    if report.records:
        r0 = report.records[0]
        it = int(r0.iterations_run)
        j["draws_per_iteration"] = int(r0.draws_used) // it if it > 0 else 0
        j["evals_per_iteration"] = int(r0.evals_used) // it if it > 0 else 0
    return _json_dump(j) + "\n"


REPLICATE_VECTORS = ("params", "prop", "diff", "mean_est", "var_est", "alpha", "delta",
                     "true_grad")
_REPLICATE_HEADER = {"params": "param", "prop": "prop", "diff": "diff", "mean_est": "mean_est",
                     "var_est": "var_est", "alpha": "alpha", "delta": "delta",
                     "true_grad": "true_grad"}


def write_replicate_csv(record, out: Union[str, IO[str]]) -> None:
    """harness.cpp:344-365: the wide per-iteration table of one replicate.
    `record` must carry the full vectors (api.run_single(..., full=True));
    the alpha columns appear only for meta runs (record.vectors['alpha']
    is None for Adam)."""
    vec = getattr(record, "vectors", None)
    if vec is None:
        raise ValueError("record has no per-iteration vectors; run with full=True")
    n_it = int(record.iterations_run)
    dim = vec["params"].shape[1] if n_it > 0 else 0
    names = [n for n in REPLICATE_VECTORS if n != "alpha" or vec.get("alpha") is not None]
    buf = io.StringIO()
    buf.write("iteration,loss,step_sq_norm")
    for n in names:
        for j in range(dim):
            buf.write(f",{_REPLICATE_HEADER[n]}_{j}")
    buf.write("\n")
    loss, ssn = record.series["loss"], record.series["step_sq_norm"]
    for i in range(n_it):
        buf.write(f"{i},{format_double(float(loss[i]))},{format_double(float(ssn[i]))}")
        for n in names:
            for x in vec[n][i]:
                buf.write("," + format_double(float(x)))
        buf.write("\n")
    text = buf.getvalue()
    if isinstance(out, str):
        with open(out, "w", newline="") as f:
            f.write(text)
    else:
        out.write(text)
