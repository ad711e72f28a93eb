# A/B: Hex8 z-sweep unrolled by 2 (tools/libtopo_u2.so) vs the product build
mkdir -p gpurun_out
for lib in "" tools/libtopo_u2.so; do
  echo "lib=${lib:-product}" >> gpurun_out/hex8_unroll.log
  TB_LIB_PATH=$lib timeout 120 python profiles/apply_once.py cfg3 >> gpurun_out/hex8_unroll.log 2>&1
  TB_LIB_PATH=$lib timeout 200 python profiles/iter_time.py cfg3 >> gpurun_out/hex8_unroll.log 2>&1
done
