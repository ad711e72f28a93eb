# 3D (cfg3) multigrid smoother: iterations and evaluation time for V(nu,nu), omega
mkdir -p gpurun_out
for nu in 1 2; do
  for om in 0.4 0.5 0.6; do
    echo "nu=$nu omega=$om cfg3: $(TB_MG_NU=$nu TB_MG_OMEGA=$om timeout 200 python profiles/mg_once.py cfg3 3 2>&1 | tail -1)" >> gpurun_out/mg_nu3d.log
  done
done
