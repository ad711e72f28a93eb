# quick timing of the 2D MG evaluation (cfg2, cfg1) and the per-phase profile (cfg2)
mkdir -p gpurun_out
for c in cfg2 cfg1; do echo "$c: $(timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/mg_quick.log; done
TB_LIB_PATH=tools/libtopo_mgprof.so timeout 200 python profiles/mg_prof.py cfg2 2>&1 | grep -A14 "rep 2" >> gpurun_out/mg_quick.log
