#!/bin/bash
# Profiling recipe for one round (run under gpurun from the repo root).
# Writes gpurun_out/: bench lines, ncu launch list, ncu --set full reports.
set -x
R=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${R}_gpu.txt
python bench.py --bitserial > gpurun_out/${R}_bench_m1.json 2> gpurun_out/${R}_bench_m1.err
python bench.py --batch 8 --no-cpu-baseline > gpurun_out/${R}_bench_m8.json 2> gpurun_out/${R}_bench_m8.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
# every launch of a few steps (cold-cache, serialised: compare shares, not absolutes)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemv|quantize|gemm" -c 40 --csv --log-file gpurun_out/${R}_launches_m1.csv \
    python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
# full sections for the 5 GEMV launches of one step
ncu --set full --import-source on --clock-control none -k regex:gemv -c 5 -o gpurun_out/${R}_gemv_m1 \
    python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemv -c 5 -o gpurun_out/${R}_gemv_m8 \
    python bench.py --batch 8 --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
