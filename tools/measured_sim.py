"""run_simulation (kvweaver/sim_engine.py:99 semantics) on the GPU backend with
CUDA-event stage times, reported as kvweaver-csv v1 rows.

    python tools/measured_sim.py > profiles/r01_measured_sim.csv

Observations are the reference workload's token-id prefixes (obs_len = 800,
no camera images), so the prefix length matches BASELINE configs[1]'s P = 800.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_14371_b200 import BackendConfig, SimConfig, WorkloadSpec  # noqa: E402
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config  # noqa: E402
from paper_2603_14371_b200.report import measured_row, write_csv  # noqa: E402


def main():
    pc = Pi05Config()
    be = Pi05Backend(pc, num_blocks=1024, measure=True)
    # the metrics read H from the SimConfig's backend_config (kvweaver/metrics.py:117-118):
    # give it the model's chunk length so f is the H = 50 action rate
    bc = BackendConfig(H=pc.H, S=pc.S)
    rows = []
    for i, (variant, n, k) in enumerate([("Unified", 30, 5), ("SharedNoBatch", 30, 5), ("Unified", 16, 1),
                                         ("Unified", 60, 10)]):
        cfg = SimConfig(variant=variant, backend_kind="Pi05", k=k, backend_config=bc,
                        workload=WorkloadSpec(pattern="OnePerFrame", default_N=n, obs_len=800, num_frames=24))
        rows.append(measured_row(f"r{i:04d}", cfg, be))
    sys.stdout.write(write_csv(rows))


if __name__ == "__main__":
    main()
