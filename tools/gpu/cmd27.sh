timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', d['value'], 'apply', d['apply']['us_per_call'], 'cold', d['apply']['cold'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg3mg_launches.csv python bench.py --precond mg --no-extras --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/cfg3mg_launches.csv 2>/dev/null | head -30
