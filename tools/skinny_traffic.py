"""DRAM traffic of the skinny GEMM class (bench.py's headline roofline kernel):
for each decode / denoise projection at the frame's plan (policy split-K, the
bench's epilogue mode), one ncu pass with dram__bytes_{read,write}.sum over the
GEMM launch and its split reduce (L2 flushed before each launch, as bench.py
times them).  Writes gpurun_out/skinny_traffic.json: per-shape traffic vs the
algorithmic bytes, and the per-frame class total (launches per frame weighted).

    python tools/skinny_traffic.py            # drives ncu, one pass per shape
    python tools/skinny_traffic.py N K T MODE SPLITS   # child: 3 flushed launches"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(n, kk, t, mode, splits):
    import torch
    import bench
    fn, keep = bench.gemm_launcher(n, kk, t, mode, splits)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        flush.zero_()
        fn()
    torch.cuda.synchronize()


def shapes():
    from paper_2603_14371_b200.pi05 import Pi05Config
    import bench
    cfg = Pi05Config()
    llm, exp, _ = bench.projections(cfg)
    names, modes = ("qkv", "o", "gate_up", "down"), (1, 2, 3, 2)
    k, m, r = 5, 6, 1
    out = [(f"decode.{nm}", n, kk, m, md, k * cfg.depth) for nm, (n, kk), md in zip(names, llm, modes)]
    out.append(("decode.lm_head", cfg.vocab, cfg.width, m, 0, k))
    out += [(f"denoise.{nm}", n, kk, cfg.H * r, md, cfg.S * cfg.depth) for nm, (n, kk), md in zip(names, exp, modes)]
    return out


def parse(path):
    """{launch id: {metric: bytes}} of the last launch group (GEMM + reduce) in an ncu csv."""
    lines = [l for l in open(path) if l.startswith('"')]
    per = {}
    for r in csv.DictReader(lines):
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                 "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
        per.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"].split("(")[0]})[r["Metric Name"]] = v * scale
    return per


def main():
    import bench
    res, tot_alg, tot_traffic = {}, 0.0, 0.0
    for name, n, kk, t, mode, per_frame in shapes():
        sp = bench.policy_splits(1, n, kk)
        log = os.path.join(ROOT, "gpurun_out", f"skinny_{name}.csv")
        subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                        "-k", "regex:gemm_kernel|splitk", "--csv", "--log-file", log, sys.executable,
                        os.path.abspath(__file__), str(n), str(kk), str(t), str(mode), str(sp)],
                       check=True, capture_output=True)
        launches = parse(log)
        per_group = 2 if sp > 1 else 1
        last = [launches[i] for i in sorted(launches)[-per_group:]]
        traffic = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in last)
        alg = n * kk * 2 + t * kk * 2 + t * (n // 2 if mode == 3 else n) * (4 if mode in (0, 2) else 2)
        res[name] = {"shape": f"{n}x{kk} T={t} splits={sp}", "algorithmic_bytes": alg, "traffic_bytes": traffic,
                     "traffic_over_algorithmic": traffic / alg, "launches_per_frame": per_frame,
                     "kernels": [l["kernel"] for l in last],
                     "ncu_us": sum(l.get("gpu__time_duration.sum", 0) for l in last)}
        tot_alg += alg * per_frame
        tot_traffic += traffic * per_frame
    out = {"skinny_class": {"traffic_bytes_per_frame": tot_traffic, "algorithmic_bytes_per_frame": tot_alg,
                            "traffic_over_algorithmic": tot_traffic / tot_alg,
                            "method": "ncu dram__bytes_read.sum + dram__bytes_write.sum of each shape's GEMM "
                                      "+ split reduce, L2 flushed before the launch, x launches per frame"},
           "skinny_shapes": res}
    with open(os.path.join(ROOT, "gpurun_out", "skinny_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["skinny_class"]))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(*[int(a) for a in sys.argv[1:]])
    else:
        main()
