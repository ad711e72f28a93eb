python -m pytest tests/test_gpu_rom.py -x -q -m gpu > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
for v in variants/lib_v9.so paper_2004_05756_b200/libtopo_b200.so; do echo $v; TB_LIB_PATH=$v python profiles/gs_time.py; done > gpurun_out/gs_time.log 2>&1
cat gpurun_out/gs_time.log
python -m pytest tests -x -q -m gpu > gpurun_out/t4all.log 2>&1; tail -3 gpurun_out/t4all.log
