"""Export the `ncu --set full` captures of tools/profile_all.sh (gpurun_out/ncu_*.ncu-rep)
to profiles/ncu/<round>_<name>_{details,raw}.csv and write profiles/<round>_ncu_traffic.json
(DRAM bytes per launch of each roofline kernel; bench.py's roofline.traffic).
    python tools/ncu_export.py r01"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CAPTURES = {  # profile_all.sh report name -> (profiles name, description)
    "ncu_lm_head": ("lm_head", "gemm_sm100 (tcgen05) @ LM head 257152x2048, T=6"),
    "ncu_dn_down": ("dn_down", "gemm_sm100 (tcgen05, split-K 16) @ expert down 1024x4096, T=50"),
    "ncu_dec_down": ("dec_down", "gemm_sm100 (tcgen05, split-K 9) @ decode down 2048x16384, T=6"),
    "ncu_prefill_gu": ("prefill_gu", "gemm_wide_kernel<2> (tcgen05 cta_group::2) @ prefill gate/up 32768x2048, T=800"),
    "ncu_decode_attn": ("decode_attn", "decode attention (TMA ring) @ 256 rows x 1024 ctx"),
    "ncu_flash_tc": ("flash_tc", "flash_tc (tcgen05 attention) @ prefill P=800, 8 heads, 2 key splits"),
    "ncu_vit_attn": ("vit_attn", "vit_attn_tc (tcgen05 SigLIP attention) @ 3 images x 16 heads x 256 tokens"),
}


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True, check=True)
    return out.stdout


def main(rnd):
    traffic = {}
    for rep_name, (name, desc) in CAPTURES.items():
        rep = os.path.join(ROOT, "gpurun_out", rep_name + ".ncu-rep")
        if not os.path.exists(rep):
            print("missing", rep)
            continue
        details, raw = ncu_csv(rep, "details"), ncu_csv(rep, "raw")
        for kind, text in (("details", details), ("raw", raw)):
            with open(os.path.join(ROOT, "profiles", "ncu", f"{rnd}_{name}_{kind}.csv"), "w") as f:
                f.write(text)
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, vals = rows[0], rows[2]  # row 1 holds the units
        g = dict(zip(hdr, vals))
        num = lambda k: float(g[k].replace(",", "")) if g.get(k, "") not in ("", "n/a") else None  # noqa: E731
        units = dict(zip(hdr, rows[1]))
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
        wr *= scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
        dur = num("gpu__time_duration.sum") * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(
            units.get("gpu__time_duration.sum", "usecond"), 1.0)
        traffic[name] = {"kernel": desc, "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                         "ncu_duration_us": round(dur, 3),
                         "dram_pct_of_peak": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                         "tensor_pipe_pct_active": num(
                             "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                         "grid": g.get("launch__grid_size")}
    path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_traffic.json")
    merged = {}
    if os.path.exists(path):  # keep entries written by other tools (skinny_traffic.py's class)
        with open(path) as f:
            merged = json.load(f)
    merged.update(traffic)
    with open(path, "w") as f:
        json.dump(merged, f, indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
