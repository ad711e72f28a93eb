# graph-path iteration counts for V(nu,nu) cycles and Jacobi damping (TB_MG_NU, TB_MG_OMEGA)
mkdir -p gpurun_out
for c in cfg2 cfg1; do
  for nu in 1 2 3; do
    for om in 0.5 0.6 0.7; do
      echo "nu=$nu omega=$om $c: $(TB_NO_PERSIST=1 TB_MG_NU=$nu TB_MG_OMEGA=$om timeout 120 python profiles/mg_once.py $c 2 2>&1 | tail -1)" >> gpurun_out/mg_nu.log
    done
  done
done
