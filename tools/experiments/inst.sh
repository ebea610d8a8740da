python bench.py --skip-load --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 1 > /dev/null 2>&1
for v in "" "FDY_EXP_NOPDL=1" "FDY_EXP_RGRID=148" "FDY_EXP_RGRID=296" "FDY_EXP_RGRID=592" "FDY_EXP_RGRID=1776"; do
  echo "== $v"; env $v python tools/gpu_floor.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['best_us'],v['median_us']) for k,v in d.items() if 'materialize' in k})"
done
