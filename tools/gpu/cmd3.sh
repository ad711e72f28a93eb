ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_hex8_cg<1>|k_hex8<' -c 4 -o gpurun_out/apply_modes python profiles/apply_modes.py > gpurun_out/ncu_apply.log 2>&1
tail -2 gpurun_out/ncu_apply.log
