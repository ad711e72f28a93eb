# persistent MG-pCG solve/eval times: default smoother vs V(2,2) omega 0.6
mkdir -p gpurun_out
for c in cfg2 cfg1; do
  echo "default $c: $(timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/mg_ab.log
  echo "V22 w0.6 $c: $(TB_MG_NU=2 TB_MG_OMEGA=0.6 timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/mg_ab.log
  echo "V22 w0.7 $c: $(TB_MG_NU=2 TB_MG_OMEGA=0.7 timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/mg_ab.log
  echo "V11 w0.8 $c: $(TB_MG_NU=1 TB_MG_OMEGA=0.8 timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/mg_ab.log
done
TB_LIB_PATH=tools/libtopo_mgprof.so timeout 200 python profiles/mg_prof.py cfg2 2>&1 | grep -A14 "rep 2" >> gpurun_out/mg_ab.log
