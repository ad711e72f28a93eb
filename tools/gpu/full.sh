# full checkpoint: GPU tests, default bench (headline + extras), smoke, ncu of the sweep, launch list
python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; tail -2 gpurun_out/full_tests.log
python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; tail -c 300 gpurun_out/full_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; tail -2 gpurun_out/full_smoke.log
NREP=4 ncu --set full --clock-control none --import-source on -k regex:k_hex8_cg -c 4 -o gpurun_out/full_sweep python profiles/sweep_once.py > /dev/null 2>&1
TB_PCG_NOGRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/full_launches.csv python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/full_nograph.json 2>/dev/null
echo done
