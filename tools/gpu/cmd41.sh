for v in paper_2004_05756_b200/libtopo_b200.so variants/lib_mgp_16_16.so variants/lib_mgp_8_32.so variants/lib_mgp_16_32.so; do
  for c in cfg2 cfg1; do
  TB_LIB_PATH=$v timeout 300 python bench.py --config $c --precond mg --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c mg s/eval', round(d['value']*1e3,3), 'ms its', d['config']['pcg_iterations'], 'mgpcg us', round(d['roofline']['us_per_launch'],1))"
  done
done
