set -u
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2n
mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_endpoint.py tests/test_abi.py -m gpu -x -q -k "diagnostics or abi or unreachable or goldens_small" > $o/pytest.log 2>&1; echo "pytest exit $?" >> $o/pytest.log
tail -30 $o/pytest.log
