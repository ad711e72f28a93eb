ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_mg_gj_inverse -c 2 python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 1 --warmup 3 2>&1 | grep -E "gpu__time|inst_exec"
python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2 mg s/eval', d['value'], 'e2e', d['e2e']['value'])"
python -m pytest tests/test_gpu_mg.py tests/test_gpu_cfg2.py -x -q -m gpu 2>&1 | tail -1
