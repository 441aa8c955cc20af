"""Stage times of the 1-stream frame with each stage forced onto its SM partition
(OXY_GREEN_FORCE=1) and run back to back (stage-serial frame): how fast are the decode
on 68 SMs and the denoise on 80 SMs with nothing running beside them?"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for env in ({}, {"OXY_GREEN_FORCE": "1"}):
    out = subprocess.run([sys.executable, "bench.py", "--steps", "10", "--warmup", "4", "--no-cpu-baseline"],
                         cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    print(env, "overlapped", d["stage_ms"], "stage-serial", d["stage_serial"]["stage_ms"])
