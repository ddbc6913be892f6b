S='import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get("layer"), d.get("m"), round(d["us_gemm"],1), round(d["frac_hbm"],3))'
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader
for i in 1 2; do
echo HEAD; FLEXQ_LIB=paper_2508_04405_b200/_lib/libflexq_head.so python tools/sweep.py --model llama2-70b --ms 64,128 --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep gate
echo NEW; python tools/sweep.py --model llama2-70b --ms 64,128 --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep gate
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader
