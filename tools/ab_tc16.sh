# A/B on one box: the kind::f16 batched path vs the INT8 tcgen05 path (FLEXQ_DISABLE_TC16=1)
S='import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d.get("layer"), d.get("m"), round(d["us_gemm"],1), round(d["us_fwd"],1), round(d["frac_hbm"],3))'
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader
for i in $(seq ${REPS:-2}); do
echo TC16; python tools/sweep.py --model ${MODEL:-llama2-70b} --ms ${MS:-64,128} --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep -E "${LAYERS:-gate|qkv}"
echo I8; FLEXQ_DISABLE_TC16=1 python tools/sweep.py --model ${MODEL:-llama2-70b} --ms ${MS:-64,128} --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep -E "${LAYERS:-gate|qkv}"
done
