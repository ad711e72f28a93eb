timeout 600 python -m pytest tests/test_gpu_mg.py tests/test_gpu_cfg2.py tests/test_gpu_hdm.py -x -q -m gpu 2>&1 | tail -1
for e in 0 1; do
  if [ $e = 1 ]; then export TB_MGP_UNFUSED=1; fi
  for c in cfg2 cfg1; do
  timeout 300 python bench.py --config $c --precond mg --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('unfused=$e $c mg s/eval', round(d['value']*1e3,3), 'ms its', d['config']['pcg_iterations'], 'mgpcg us', round(d['roofline']['us_per_launch'],1))"
  done
done
