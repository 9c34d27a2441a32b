"""Reference-format reports of a device run:
byte-for-byte the CSV the reference harness writes (harness.cpp:305-342),
so a user of the reference can diff outputs directly.

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
