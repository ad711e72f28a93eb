timeout 600 python bench.py --config cfg5 --no-extras --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['value'], d['roofline']['us_per_launch'], d['roofline']['frac'])"
timeout 600 python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py -q -m gpu -k "rom or cfg5 or reduced" 2>&1 | tail -2
