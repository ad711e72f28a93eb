python bench.py --no-extras --no-cpu-baseline > gpurun_out/b8_cfg3.json 2> gpurun_out/b8_cfg3.err
python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 5 > gpurun_out/b8_cfg2.json 2> gpurun_out/b8_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg2mg_launches.csv python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/cfg2mg_launches.csv | head -24
