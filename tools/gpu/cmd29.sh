TB_PCG_NOGRAPH=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_helm3d<\(bool\)1>' -s 5 -c 1 -o gpurun_out/helm3d python profiles/apply_modes.py > gpurun_out/ncu_helm.log 2>&1
tail -1 gpurun_out/ncu_helm.log
