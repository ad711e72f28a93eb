mkdir -p gpurun_out
for c in cfg2 cfg1; do
  TB_LIB_PATH=tools/libtopo_mgprof.so timeout 200 python profiles/mg_prof.py $c 2>&1 | grep -A14 "rep 2" >> gpurun_out/mg_prof3.log
  TB_NO_PERSIST=1 timeout 200 python profiles/mg_prof.py $c 2>&1 | grep "rep 2" | sed "s/^/graph $c /" >> gpurun_out/mg_prof3.log
done
