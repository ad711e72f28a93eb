#!/bin/bash
# A/B of the single-sweep pCG: the product build against variants/lib*.so given as arguments,
# interleaved on the same box (tb_pcg_profile per-launch events, then one timed cfg 3 solve).
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in "" "$@"; do
    echo "lib=${lib:-product} $(TB_LIB_PATH=$lib NREP=30 timeout 120 python profiles/sweep_once.py 2>&1 | tail -1)"
  done
done
for lib in "" "$@"; do
  echo "lib=${lib:-product} solve: $(TB_LIB_PATH=$lib timeout 200 python profiles/iter_time.py cfg3 2>&1 | tail -1)"
done
