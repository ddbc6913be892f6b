#!/bin/bash
# Measurement + profiling recipe for one round (run under gpurun from the repo root).
# Writes gpurun_out/<R>_*: bench lines, M sweeps, decode bench, ncu launch list and
# --set full captures of the GEMM kernels; tools/summarize_ncu.py turns them into profiles/.
set -x
R=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${R}_gpu.txt
python bench.py > gpurun_out/${R}_bench_m1.json 2> gpurun_out/${R}_bench_m1.err
python bench.py --batch 8 --no-cpu-baseline --no-extra > gpurun_out/${R}_bench_m8.json 2> gpurun_out/${R}_bench_m8.err
python bench.py --batch 32 --steps 1000 --no-cpu-baseline --no-extra > gpurun_out/${R}_bench_m32.json 2> gpurun_out/${R}_bench_m32.err
python bench.py --batch 64 --steps 500 --no-cpu-baseline --no-extra > gpurun_out/${R}_bench_m64.json 2> gpurun_out/${R}_bench_m64.err
python bench.py --batch 128 --steps 500 --no-cpu-baseline --no-extra > gpurun_out/${R}_bench_m128.json 2> gpurun_out/${R}_bench_m128.err
python bench.py --batch 256 --steps 300 --no-cpu-baseline --no-extra > gpurun_out/${R}_bench_m256.json 2> gpurun_out/${R}_bench_m256.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
for mdl in llama2-7b llama2-13b llama2-70b; do
  python tools/sweep.py --model $mdl --ms 1,2,4,8,16,32,64,128,256 > gpurun_out/${R}_sweep_${mdl}.jsonl 2> gpurun_out/${R}_sweep_${mdl}.err
done
python tools/decode_bench.py --model 7b --batches 1,2,4,8 --steps 128 --warmup 32 > gpurun_out/${R}_decode_7b.jsonl 2> gpurun_out/${R}_decode_7b.err
# every launch of a few steps (cold-cache, serialised: compare shares, not absolutes)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemv|quantize|gemm" -c 40 --csv --log-file gpurun_out/${R}_launches_m1.csv \
    python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extra --no-bitserial > /dev/null 2>&1
# full sections for the 5 GEMM launches of one step; exported to CSV on the box (the
# reports themselves would exceed gpurun's 64 MiB copy-back), one small report kept
for m in 1 8 32 64 128; do
  ncu --set full --import-source on --clock-control none -k regex:"gemv|gemm_tc" -c 5 -o /tmp/${R}_gemm_m$m \
      python bench.py --batch $m --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extra --no-bitserial > /dev/null 2>&1
  ncu -i /tmp/${R}_gemm_m$m.ncu-rep --page raw --csv > gpurun_out/${R}_gemm_m${m}_raw.csv
  ncu -i /tmp/${R}_gemm_m$m.ncu-rep --page details --csv > gpurun_out/${R}_gemm_m${m}_details.csv
done
ncu --set full --import-source on --clock-control none -k regex:"gemv" -c 1 -o gpurun_out/${R}_gemv_m1_one \
    python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-extra --no-bitserial > /dev/null 2>&1
du -sh gpurun_out; ls -la gpurun_out
