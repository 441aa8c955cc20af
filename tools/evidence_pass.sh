set -x
bash tools/profile_all.sh > gpurun_out/profile_all.log 2>&1
python tools/ncu_export.py r02 > gpurun_out/ncu_export.log 2>&1
python tools/skinny_traffic.py > gpurun_out/skinny.log 2>&1
mkdir -p gpurun_out/export
cp -r profiles/ncu gpurun_out/export/; cp profiles/r02_ncu_traffic.json gpurun_out/export/
rm -f gpurun_out/*.ncu-rep
python tools/config_sweep.py all > gpurun_out/config_sweep.jsonl 2> gpurun_out/config_sweep.err
du -sh gpurun_out
