cd $GRAFT_REPO_ROOT
o=gpurun_out/acc2.log; : > $o
# 1) pure reference (CPU, SuperLU): ssbeam MMA reference history (cached for step 2) and its TR run
ACC_DROPIN=0 timeout 1500 python tools/gpu/acc_diag.py ssbeam rom-tr-res >> $o 2>&1
# 2) the reference's acceptance criteria 6-8 on the drop-in, MMA histories from the reference's cache
cd baseline/_ref/romtopt_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -p dropin_plugin -p no:cacheprovider -o addopts= test_acceptance.py -s -rA 2>&1 | tail -80 >> $GRAFT_REPO_ROOT/$o
