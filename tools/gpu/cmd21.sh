for c in cfg1 cfg2; do for m in 300 600 1200 2500; do
  TB_MG_MIN_DOFS=$m timeout 300 python bench.py --config $c --precond mg --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c min_dofs=$m s/eval', round(d['value']*1e3,3), 'ms its', d['config']['pcg_iterations'], 'mgpcg us', round(d['roofline']['us_per_launch'],1))"
done; done
