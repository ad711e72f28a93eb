for v in paper_2004_05756_b200/libtopo_b200.so variants/lib_apply3.so; do echo $v; TB_LIB_PATH=$v python profiles/apply_once.py cfg3; TB_LIB_PATH=$v python profiles/apply_once.py cfg5; done
TB_LIB_PATH=variants/lib_apply3.so timeout 600 python -m pytest tests/test_gpu_3d.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -1
