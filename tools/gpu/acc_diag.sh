cd $GRAFT_REPO_ROOT
o=gpurun_out/acc_diag.log; : > $o
ACC_DROPIN=1 timeout 900 python tools/gpu/acc_diag.py ssbeam rom-tr-res >> $o 2>&1
ACC_DROPIN=1 TB_DROPIN_RTOL=-1e-14 timeout 900 python tools/gpu/acc_diag.py ssbeam rom-tr-res >> $o 2>&1
ACC_DROPIN=1 TB_DROPIN_PRECOND=mg timeout 900 python tools/gpu/acc_diag.py ssbeam rom-tr-res >> $o 2>&1
ACC_DROPIN=0 timeout 1200 python tools/gpu/acc_diag.py ssbeam rom-tr-res >> $o 2>&1
