# A/B of the grid barrier variants: per-solve times of the persistent 2D kernels (MG + Jacobi)
mkdir -p gpurun_out
for c in cfg2 cfg1; do
  echo "mg $c: $(timeout 120 python profiles/mg_once.py $c 4 2>&1 | tail -1)" >> gpurun_out/barrier_ab.log
  echo "jacobi $c: $(TB_PRECOND=jacobi timeout 120 python profiles/iter_time.py $c 2>&1 | tail -1)" >> gpurun_out/barrier_ab.log
done
