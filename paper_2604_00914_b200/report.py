"""RunReport: the machine-readable record of one solve, and the solve flow that emits it.

Mirrors proj/include/adapoly/run_report.hpp:10-27 / proj/src/run_report.cpp:7-148:
the same document (config echo, matrix metadata, result summary, per-iteration
table, stage timings) with the same field names, parsed back by
`run_report_from_json`, and `dump_report` writes it byte-compatibly with the
reference's `nlohmann::json::dump(2)`: keys sorted, two-space indent, numbers in
nlohmann's shortest-round-trip format, a trailing newline. GPU runs add one
optional top-level "device" object (ignored by the reference's reader).

`run_solve` restates the `solve` subcommand's flow (proj/src/cli.cpp:152-196)
as a library call: load a symmetric Matrix Market file, solve on the GPU,
build the report, optionally write the eigenvector table; it returns the
reference's exit codes (0 converged, 1 input error, 2 not converged).
"""
from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

from .filter import SpectrumBounds
from .solver import IterationRecord, SolveResult, SolverConfig, StageTimings

EXIT_OK, EXIT_INPUT_ERROR, EXIT_NOT_CONVERGED = 0, 1, 2


@dataclass
class RunReport:
    config: SolverConfig = field(default_factory=SolverConfig)
    threads: int = 0
    matrix_path: str = ""
    n: int = 0
    nnz: int = 0
    result: SolveResult | None = None
    device: dict | None = None  # GPU fields (name, SMs, kernel launches, library); None -> omitted


def _num(x):
    return None if x is None else x


def to_json(report: RunReport) -> dict:
    """to_json (run_report.cpp:7-82)."""
    c = report.config
    cfg = {
        "interval_a": float(c.interval_a), "interval_b": float(c.interval_b), "tau_c": float(c.tau_c),
        "tau_a": float(c.tau_a), "m": float(c.m), "C": float(c.c), "k_multiplier": float(c.k_multiplier),
        "mu": float(c.mu), "max_iter": int(c.max_iter), "lanczos_steps": int(c.lanczos_steps),
        "trace_probes": int(c.trace_probes), "rng_seed": int(c.rng_seed),
        "p_override": None if c.p_override is None else int(c.p_override),
        "tile_ti": None if getattr(c, "tile_ti", None) is None else int(c.tile_ti),
        "tile_tk": None if getattr(c, "tile_tk", None) is None else int(c.tile_tk),
        "threads": int(report.threads),
    }
    r = report.result
    result = {
        "converged": bool(r.converged), "dense_fallback": bool(r.dense_fallback),
        "eigenvalues": [float(v) for v in np.asarray(r.eigenvalues, np.float64).ravel()],
        "iterations": int(r.iterations), "spmv_total": int(r.spmv_total), "avg_degree": float(r.avg_degree),
        "max_residual": float(r.max_residual), "e_estimate": float(r.e_estimate),
        "subspace_dim": int(r.subspace_dim),
        "spectrum_bounds": {"lambda_min": float(r.bounds.lambda_min), "lambda_max": float(r.bounds.lambda_max)},
        "degree_history": [int(d) for d in r.degree_history],
    }
    table = [{
        "iteration": int(h.iteration), "degree": int(h.degree), "active_width": int(h.active_width),
        "e_in_interval": int(h.e_in_interval), "n_locked": int(h.n_locked_total),
        "max_residual": float(h.max_residual), "spmv_filter": int(h.spmv_filter),
        "spmv_residual": int(h.spmv_residual),
    } for h in r.history]
    t = r.timings
    timings = {"setup": float(t.setup), "filter": float(t.filter), "orth": float(t.orth),
               "rayleigh_ritz": float(t.rayleigh_ritz), "residuals": float(t.residuals), "other": float(t.other)}
    doc = {
        "config": cfg,
        "matrix": {"path": report.matrix_path, "n": int(report.n), "nnz": int(report.nnz)},
        "result": result,
        "iteration_table": table,
        "timings": timings,
    }
    if report.device is not None:
        doc["device"] = dict(report.device)
    return doc


def run_report_from_json(j: dict) -> RunReport:
    """run_report_from_json (run_report.cpp:84-144); KeyError on a missing field, like json::at."""
    cfg = j["config"]
    c = SolverConfig(
        interval_a=float(cfg["interval_a"]), interval_b=float(cfg["interval_b"]), tau_c=float(cfg["tau_c"]),
        tau_a=float(cfg["tau_a"]), m=float(cfg["m"]), c=float(cfg["C"]), k_multiplier=float(cfg["k_multiplier"]),
        mu=float(cfg["mu"]), max_iter=int(cfg["max_iter"]), lanczos_steps=int(cfg["lanczos_steps"]),
        trace_probes=int(cfg["trace_probes"]), rng_seed=int(cfg["rng_seed"]),
        p_override=None if cfg["p_override"] is None else int(cfg["p_override"]),
        tile_ti=None if cfg["tile_ti"] is None else int(cfg["tile_ti"]),
        tile_tk=None if cfg["tile_tk"] is None else int(cfg["tile_tk"]))
    res = j["result"]
    history = [IterationRecord(iteration=int(row["iteration"]), degree=int(row["degree"]),
                               active_width=int(row["active_width"]), e_in_interval=int(row["e_in_interval"]),
                               n_locked_total=int(row["n_locked"]), max_residual=_f(row["max_residual"]),
                               spmv_filter=int(row["spmv_filter"]), spmv_residual=int(row["spmv_residual"]),
                               orth_error=-1.0)
               for row in j["iteration_table"]]
    t = j["timings"]
    r = SolveResult(
        eigenvalues=np.array([_f(v) for v in res["eigenvalues"]], np.float64),
        eigenvectors=np.zeros((int(j["matrix"]["n"]), 0)),
        converged=bool(res["converged"]), dense_fallback=bool(res["dense_fallback"]),
        iterations=int(res["iterations"]), spmv_total=int(res["spmv_total"]), avg_degree=_f(res["avg_degree"]),
        max_residual=_f(res["max_residual"]), degree_history=[int(d) for d in res["degree_history"]],
        history=history,
        bounds=SpectrumBounds(_f(res["spectrum_bounds"]["lambda_min"]), _f(res["spectrum_bounds"]["lambda_max"])),
        e_estimate=_f(res["e_estimate"]), subspace_dim=int(res["subspace_dim"]),
        timings=StageTimings(setup=_f(t["setup"]), filter=_f(t["filter"]), orth=_f(t["orth"]),
                             rayleigh_ritz=_f(t["rayleigh_ritz"]), residuals=_f(t["residuals"]), other=_f(t["other"])))
    return RunReport(config=c, threads=int(cfg["threads"]), matrix_path=str(j["matrix"]["path"]),
                     n=int(j["matrix"]["n"]), nnz=int(j["matrix"]["nnz"]), result=r, device=j.get("device"))


def _f(v) -> float:
    return math.nan if v is None else float(v)  # nlohmann writes non-finite doubles as null


# ------------------------------------------------------------------ dump(2) ---
def format_double(x: float) -> str:
    """A double the way nlohmann::json serialises it (dtoa_impl::format_buffer, min_exp -4, max_exp 15)."""
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    s = repr(abs(x))  # shortest round-trip digits
    mant, _, exp = s.partition("e")
    ip, _, fp = mant.partition(".")
    digits = ip + fp
    point = len(ip) + (int(exp) if exp else 0)
    stripped = digits.lstrip("0")
    point -= len(digits) - len(stripped)
    digits = stripped.rstrip("0") or "0"
    k, n = len(digits), point
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    body = digits if k == 1 else digits[0] + "." + digits[1:]
    return sign + body + "e" + ("-" if e < 0 else "+") + ("%02d" % abs(e))


def _escape(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif o < 0x20:
            out.append("\\u%04x" % o)
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def _dump(v, level: int, out: list) -> None:
    pad = "  "
    if v is None:
        out.append("null")
    elif isinstance(v, bool):
        out.append("true" if v else "false")
    elif isinstance(v, (int, np.integer)):
        out.append(str(int(v)))
    elif isinstance(v, (float, np.floating)):
        out.append(format_double(float(v)))
    elif isinstance(v, str):
        out.append(_escape(v))
    elif isinstance(v, dict):
        if not v:
            out.append("{}")
            return
        out.append("{\n")
        items = sorted(v.items())  # nlohmann::json objects are std::map: keys in sorted order
        for i, (key, val) in enumerate(items):
            out.append(pad * (level + 1) + _escape(key) + ": ")
            _dump(val, level + 1, out)
            out.append(",\n" if i + 1 < len(items) else "\n")
        out.append(pad * level + "}")
    elif isinstance(v, (list, tuple)):
        if not v:
            out.append("[]")
            return
        out.append("[\n")
        for i, val in enumerate(v):
            out.append(pad * (level + 1))
            _dump(val, level + 1, out)
            out.append(",\n" if i + 1 < len(v) else "\n")
        out.append(pad * level + "]")
    else:
        raise TypeError(f"cannot serialise {type(v).__name__}")


def dumps(doc) -> str:
    out: list = []
    _dump(doc, 0, out)
    return "".join(out)


def dump_report(report: RunReport) -> str:
    """dump_report (run_report.cpp:146-148): fixed layout, identical reports give identical bytes."""
    return dumps(to_json(report)) + "\n"


# -------------------------------------------------------------- solve flow ---
def resolved_thread_count(threads: int | None = None) -> int:
    """cli.cpp resolved_thread_count: explicit value, else ADAPOLY_THREADS, else the host's core count."""
    if threads is not None and threads > 0:
        return int(threads)
    try:
        v = int(os.environ.get("ADAPOLY_THREADS", ""))
        if v > 0:
            return v
    except ValueError:
        pass
    return os.cpu_count() or 1


def write_eigenvectors(path: str, vectors: np.ndarray) -> None:
    """write_eigenvectors (cli.cpp:102-114): 'rows cols' then one row per line, 17 significant digits."""
    try:
        fh = open(path, "w")
    except OSError:
        from ._native import ConfigError
        raise ConfigError("cannot open eigenvector file: " + path) from None
    with fh:
        v = np.asarray(vectors)
        fh.write(f"{v.shape[0]} {v.shape[1]}\n")
        for row in v:
            fh.write(" ".join(_g17(x) for x in row) + "\n")


def _g17(x: float) -> str:
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    if math.isnan(x):
        return "nan"
    return "%.17g" % x


def run_solve(matrix_path: str, config: SolverConfig, ctx=None, threads: int | None = None,
              eigenvectors_path: str | None = None, output=None, err=None) -> tuple[int, RunReport | None]:
    """The `solve` flow (cli.cpp:152-196) on the GPU: returns (exit code, report).

    The report text (dump_report) is written to `output` (a path, a file object, or None for
    nothing); errors go to `err` as 'error: <message>' with exit code 1.
    """
    from . import operator as op
    from ._native import AdpError, ConfigError, lib
    from .solver import solve
    from .sparse import read_matrix_market

    err = sys.stderr if err is None else err
    try:
        a = read_matrix_market(matrix_path)
        if a.n_rows != a.n_cols or not a.is_symmetric():
            raise ConfigError(f"matrix '{matrix_path}' is not symmetric")
        ctx = ctx or op.default_context()
        dev = op.DeviceCsr(a, ctx)
        launches0 = ctx.launch_count
        result = solve(dev, config)
        report = RunReport(config=config, threads=resolved_thread_count(threads), matrix_path=matrix_path,
                           n=a.n_rows, nnz=a.nnz, result=result,
                           device=_device_info(ctx, ctx.launch_count - launches0))
        if result.dense_fallback:
            err.write("warning: subspace dimension reached the problem size; used the dense eigensolver path\n")
        if eigenvectors_path:
            write_eigenvectors(eigenvectors_path, result.eigenvectors)
        text = dump_report(report)
        if isinstance(output, str):
            with open(output, "w") as fh:
                fh.write(text)
        elif output is not None:
            output.write(text)
        return (EXIT_OK if result.converged else EXIT_NOT_CONVERGED), report
    except (AdpError, OSError, ValueError) as e:
        err.write(f"error: {e}\n")
        return EXIT_INPUT_ERROR, None


def _device_info(ctx, launches: int) -> dict:
    info = {"library": "libadp_b200 (sm_100a)", "kernel_launches": int(launches), "device_index": int(ctx.device)}
    try:
        import torch

        if torch.cuda.is_available():
            p = torch.cuda.get_device_properties(ctx.device)
            info["name"] = p.name
            info["sm_count"] = int(p.multi_processor_count)
    except Exception:
        pass
    return info
