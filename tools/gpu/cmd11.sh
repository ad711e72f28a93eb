ncu --set full --clock-control none --import-source on -k regex:k_mg_gj_inverse -c 1 -o gpurun_out/gj python bench.py --config cfg2 --precond mg --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_gj.log 2>&1
tail -2 gpurun_out/ncu_gj.log
