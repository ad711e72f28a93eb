# the reference's own acceptance criteria 7 and 8 on the drop-in classes (diagnostic, long)
cd baseline/_ref/romtopt_tests
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -p dropin_plugin -p no:cacheprovider -o addopts= test_acceptance.py -k "${ACC_K:-criterion_8 or criterion_7}" -x -s 2>&1 | tail -60 > $GRAFT_REPO_ROOT/gpurun_out/acc78${ACC_TAG}.log
