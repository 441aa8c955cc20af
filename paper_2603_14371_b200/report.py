"""CSV v1 metrics rows for measured-latency runs.

The reference writes one ``kvweaver-csv v1`` row per simulation
(``kvweaver/cli.py:38-44`` columns, ``kvweaver/cli.py:80-101`` values, the
speedup column from an IsolatedSequential twin, ``kvweaver/cli.py:73-77``).
Its CLI is out of scope here; this module keeps the row schema so a run of
``run_simulation`` on the GPU backend — whose traces carry CUDA-event stage
microseconds instead of priced ones — lands in the same report format as the
reference's cost-model sweeps.
"""

from __future__ import annotations

import csv
import io
from dataclasses import replace

from .metrics import speedup, summarize
from .sim_engine import SimConfig, run_simulation
from .workload import generate_arrivals

__all__ = ["CSV_COLUMNS", "CSV_VERSION_COMMENT", "CSV_NOTE_COMMENT", "csv_row", "measured_row",
           "speedup_vs_isolated", "write_csv"]

CSV_COLUMNS = [
    "run_id", "variant", "backend", "N", "k", "H", "S", "lambda", "pattern",
    "seed", "frames", "f_per_request_hz", "f_aggregate_hz", "tau_tok_per_s",
    "avg_batch", "deadline_miss_rate", "warmup_frames", "speedup_vs_isolated",
]
CSV_VERSION_COMMENT = "# kvweaver-csv v1"
CSV_NOTE_COMMENT = "# avg_batch is the token-weighted mean batch size"


def _fmt(x: float) -> str:
    return f"{x:.6f}"


def _n_cell(config: SimConfig) -> str:
    wl = config.workload
    if wl.pattern == "MixedLength":
        arrivals = generate_arrivals(wl, config.backend_config.vocab)
        return _fmt(sum(a.n_tokens for a in arrivals) / len(arrivals)) if arrivals else _fmt(0.0)
    return str(wl.default_N)


def csv_row(run_id: str, config: SimConfig, result, report, spd: float, H=None, S=None) -> list[str]:
    """The v1 row (kvweaver/cli.py:80-101).  H / S default to the config's
    backend_config; GPU runs pass the model's own chunk length and step count."""
    wl = config.workload
    return [run_id, config.variant, config.backend_kind, _n_cell(config), str(config.k),
            str(H if H is not None else config.backend_config.H),
            str(S if S is not None else config.backend_config.S), _fmt(wl.arrivals_per_frame), wl.pattern,
            str(wl.seed), str(len(result.traces)), _fmt(report.per_request_action_freq),
            _fmt(report.action_freq_hz), _fmt(report.token_throughput), _fmt(report.avg_batch_size),
            _fmt(report.deadline_miss_rate), str(report.warmup_frames), _fmt(spd)]


def speedup_vs_isolated(config: SimConfig, report) -> float:
    """Speedup column: f of this run over its IsolatedSequential twin (kvweaver/cli.py:73-77)."""
    if config.variant == "IsolatedSequential":
        return 1.0
    twin = replace(config, variant="IsolatedSequential")
    return speedup(report, summarize(run_simulation(twin), twin))


# the reference CLI's private names for the same two functions (kvweaver/cli.py:73-101)
_speedup_vs_isolated = speedup_vs_isolated
_csv_row = csv_row


def measured_row(run_id: str, config: SimConfig, backend) -> list[str]:
    """Run ``config`` and its IsolatedSequential twin on one (measuring) backend
    and return the v1 row; frame times are the backend's CUDA-event stage times."""
    result = run_simulation(config, backend=backend)
    report = summarize(result, config)
    if config.variant == "IsolatedSequential":
        spd = 1.0
    else:
        twin = replace(config, variant="IsolatedSequential")
        spd = speedup(report, summarize(run_simulation(twin, backend=backend), twin))
    cfg = backend.config
    return csv_row(run_id, config, result, report, spd, H=getattr(cfg, "H", None), S=getattr(cfg, "S", None))


def write_csv(rows, fh=None) -> str:
    """The v1 file text (version + note comment lines, header, rows)."""
    out = fh or io.StringIO()
    out.write(CSV_VERSION_COMMENT + "\n")
    out.write(CSV_NOTE_COMMENT + "\n")
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    w.writerows(rows)
    return out.getvalue() if fh is None else ""
