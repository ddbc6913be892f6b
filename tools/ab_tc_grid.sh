# A/B of the tcgen05 stream-K grid (FLEXQ_TC_MIN_UNITS, FLEXQ_TC_ALIGN): GEMM-alone sweeps
# (7B/13B/70B, M = 64/128/256) and the 70B bench step at M = 64/128
S='import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if "us_gemm" in d: print(d.get("model")[-3:], d.get("layer"), d.get("m"), d.get("kernel"), round(d["us_gemm"],1))'
B='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench M=%d: %.1f us/step %.1f TOPS" % (d["config"]["batch"], d["ms_per_step"]*1e3, d["value"]))'
for cfg in ${CFGS:-default FLEXQ_TC_ALIGN=1}; do
  echo "== $cfg"
  for md in llama2-7b llama2-13b llama2-70b; do
    env $([ "$cfg" = default ] || echo $cfg) python tools/sweep.py --model $md --ms ${MS:-64,128,256} --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep -E "${LAYERS:-q_proj|qkv|gate|down}"
  done
  for m in 64 128; do
    env $([ "$cfg" = default ] || echo $cfg) python bench.py --batch $m --steps 300 --no-cpu-baseline --no-extra --no-bitserial 2>/dev/null | python -c "$B"
  done
done
