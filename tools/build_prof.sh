#!/bin/bash
# Debug build with per-phase %globaltimer probes in the persistent 2D pCG kernel.
set -e
cd "$(dirname "$0")/../paper_2004_05756_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -Xcompiler -fPIC -shared \
  -lcusolver -DTB_CGCG_PROF -o ../../tools/libtopo_prof.so *.cu
# ablation build: TB_CGCG_DBG bits skip the barrier (1), the operator (2) or the halo (4); no probes
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -Xcompiler -fPIC -shared \
  -lcusolver -DTB_CGCG_ABL -o ../../tools/libtopo_abl.so *.cu
# persistent 2D multigrid pCG with per-phase %globaltimer sums (tb_mgp_prof_read)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -Xcompiler -fPIC -shared \
  -lcusolver -DTB_MGP_PROF -o ../../tools/libtopo_mgprof.so *.cu
