mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_mle.py tests/test_abi_cpu.py -x -q -m gpu > gpurun_out/pytest_mle.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_mle.log
HMGP_STATS=1 timeout 600 python scripts/bench_trunc.py 1 2 256,256,0,64 256,256,0,128 256,256,0,192 512,512,0,128 512,512,0,192 1024,1024,0,192 2048,2048,0,192 > gpurun_out/trunc_wide.txt 2>&1
echo "trunc rc=$?" >> gpurun_out/trunc_wide.txt
