"""Fit the reference's cost model to this B200 and run the
reference's cost-model sweeps with the fitted constants.

    python tools/calibrate_cost.py > profiles/r01_cost_calibration.json

Prints one JSON object: the stage samples, the fitted CostModelParams, the
closed-form Unified vs IsolatedSequential speedup at N=30, k=5 (compare with the
measured 3.0x of profiles/r01_config_sweep.jsonl), and the N / k sweeps of
tests/test_acceptance.py:145-200 re-run through run_simulation(CostModel).
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_14371_b200 import SimConfig, WorkloadSpec, run_simulation, summarize, speedup  # noqa: E402
from paper_2603_14371_b200.calibrate import (closed_form_speedup, fit_cost_params,  # noqa: E402
                                             measure_stage_samples)


def sweep(params, n, k, frames=60):
    def cfg(variant):
        return SimConfig(variant=variant, backend_kind="CostModel", cost_params=params, k=k,
                         workload=WorkloadSpec(pattern="OnePerFrame", default_N=n, obs_len=800, num_frames=frames))
    uni, iso = cfg("Unified"), cfg("IsolatedSequential")
    return speedup(summarize(run_simulation(uni), uni), summarize(run_simulation(iso), iso))


def main():
    from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config
    be = Pi05Backend(Pi05Config(), num_blocks=512)
    samples = measure_stage_samples(be)
    params = fit_cost_params(samples["prefill"], samples["denoise"], samples["decode"])
    out = {
        "samples_us": samples,
        "fitted": dataclasses.asdict(params),
        "closed_form_speedup_N30_k5": closed_form_speedup(params, 30, 5, 800, 10),
        "sweep_N_k5": {n: sweep(params, n, 5) for n in (5, 10, 20, 30, 40)},
        "sweep_k_N30": {k: sweep(params, 30, k) for k in (1, 2, 5, 10, 15, 30)},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
