S='import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if "us_gemm" in d and d["layer"] in ("qkv_proj","o_proj","gate_proj","down_proj"): print(d.get("model")[-3:], d.get("layer"), d.get("m"), d.get("kernel"), round(d["us_gemm"],1))'
B='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench M=%d: %.1f us/step %.1f TOPS" % (d["config"]["batch"], d["ms_per_step"]*1e3, d["value"]))'
for lib in sm100a head; do
  echo "== $lib"
  FLEXQ_LIB=paper_2508_04405_b200/_lib/libflexq_$lib.so python tools/sweep.py --model llama2-70b --ms 64,128,256 --no-mma --no-cublas 2>/dev/null | python -c "$S"
  FLEXQ_LIB=paper_2508_04405_b200/_lib/libflexq_$lib.so python tools/sweep.py --model llama2-13b --ms 64,128 --no-mma --no-cublas 2>/dev/null | python -c "$S" | grep -E "gate|down"
  for m in 64 128 256; do FLEXQ_LIB=paper_2508_04405_b200/_lib/libflexq_$lib.so python bench.py --batch $m --steps 300 --no-cpu-baseline --no-extra --no-bitserial 2>/dev/null | python -c "$B"; done
done
