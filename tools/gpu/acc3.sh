cd $GRAFT_REPO_ROOT/baseline/_ref/romtopt_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT
o=$GRAFT_REPO_ROOT/gpurun_out/acc3.log; : > $o
for v in "TB_DROPIN_PRECOND=mg" "TB_DROPIN_RTOL=-1e-14" "TB_DROPIN_PRECOND=mg TB_DROPIN_RTOL=-1e-14"; do
  echo "== $v" >> $o
  env $v timeout 900 python -m pytest -q -p dropin_plugin -p no:cacheprovider -o addopts= test_acceptance.py -k criterion_8 -s 2>&1 | grep -E "criterion 8|AssumptionViolation|passed|failed" | head -5 >> $o
done
