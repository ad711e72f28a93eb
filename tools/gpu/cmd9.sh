ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:k_hex8_cg<\(int\)1>' -c 2 -o gpurun_out/apply_pitched python profiles/apply_modes.py > gpurun_out/ncu_apply2.log 2>&1
tail -2 gpurun_out/ncu_apply2.log
