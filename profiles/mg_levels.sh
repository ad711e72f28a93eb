# iterations and solve time of the 2D MG path for several coarsest-level sizes (TB_MG_MIN_DOFS)
mkdir -p gpurun_out
for c in cfg2 cfg1; do
  for m in 128 600 1200 5000; do
    echo "min_dofs=$m $c: $(TB_MG_MIN_DOFS=$m timeout 120 python profiles/mg_once.py $c 3 2>&1 | tail -1)" >> gpurun_out/mg_levels.log
  done
done
