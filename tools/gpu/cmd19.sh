timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/t19.log
cd $GRAFT_REPO_ROOT/baseline/_ref/romtopt_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -p dropin_plugin -p no:cacheprovider -o addopts= test_acceptance.py -s -rA 2>&1 | grep -E "^\[criterion|PASSED|FAILED|passed|failed|Error" > $GRAFT_REPO_ROOT/gpurun_out/acc19.log
