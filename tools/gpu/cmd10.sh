for v in paper_2004_05756_b200/libtopo_b200.so variants/lib_hy16.so; do echo $v; TB_LIB_PATH=$v NREP=50 python profiles/sweep_once.py; TB_LIB_PATH=$v python profiles/apply_once.py cfg3; done
TB_LIB_PATH=variants/lib_hy16.so python -m pytest tests/test_gpu_3d.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -2
