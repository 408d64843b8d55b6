set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2h
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_endpoint.py -m gpu -x -q > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -40 $o/pytest.log
