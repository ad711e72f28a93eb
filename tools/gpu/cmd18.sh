timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_fullsize.py tests/test_slab.py tests/test_gpu_cfg2.py -x -q -m gpu 2>&1 | tail -3
for e in 0 1; do
  if [ $e = 1 ]; then export TB_HELM3D_GENERIC=1; fi
  timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('generic=$e cfg3 s/eval', d['value'], 'e2e', d['e2e']['value'], 'sweep us', d['roofline']['us_per_launch'], d['clocks']['sm_mhz'])"
done
