NREP=1 ncu --set full --clock-control none --import-source on -k regex:k_rom_fused -c 1 -o gpurun_out/romfused python profiles/rom_once.py > gpurun_out/ncu_rf.log 2>&1
tail -2 gpurun_out/ncu_rf.log
