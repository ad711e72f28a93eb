timeout 300 python -m pytest tests/test_gpu_mg.py tests/test_gpu_cfg2.py -x -q -m gpu 2>&1 | tail -2
for e in 0 1; do
  if [ $e = 1 ]; then export TB_MGP_NOCLUSTER=1; fi
  timeout 300 python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nocluster=$e cfg2 mg s/eval', d['value'], 'e2e', d['e2e']['value'], 'its', d['config']['pcg_iterations'], 'us/launch', d['roofline']['us_per_launch'])"
  timeout 300 python bench.py --config cfg1 --precond mg --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nocluster=$e cfg1 mg s/eval', d['value'], 'its', d['config']['pcg_iterations'], 'us/launch', d['roofline']['us_per_launch'])"
done
