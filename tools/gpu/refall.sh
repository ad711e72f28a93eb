cd $GRAFT_REPO_ROOT/baseline/_ref/romtopt_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -p dropin_plugin -p no:cacheprovider -o addopts= . --ignore=test_acceptance.py -rf 2>&1 | tail -15 > $GRAFT_REPO_ROOT/gpurun_out/refall.log
