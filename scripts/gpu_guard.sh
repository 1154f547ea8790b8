cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/guard
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k guard_bands > gpurun_out/guard/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/guard/pytest.log
tail -30 gpurun_out/guard/pytest.log
