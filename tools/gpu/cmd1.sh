set -x
for v in variants/lib_v9.so paper_2004_05756_b200/libtopo_b200.so; do TB_LIB_PATH=$v NREP=50 python profiles/sweep_once.py; done
python -m pytest tests/test_gpu_3d.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
NREP=4 ncu --set full --clock-control none --import-source on -k regex:k_hex8_cg -c 4 -o gpurun_out/sweep_lag python profiles/sweep_once.py > gpurun_out/ncu_lag.log 2>&1
tail -3 gpurun_out/ncu_lag.log
