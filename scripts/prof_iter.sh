# one build->measure iteration: GPU parity tests, truncation micro-bench, C3 phases
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/iter_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
HMGP_STATS=1 timeout 300 python scripts/bench_trunc.py 2 256,256,0,96 256,256,0,192 512,512,0,192 1024,1024,0,192 > gpurun_out/iter_trunc.txt 2>&1
timeout 300 python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 > gpurun_out/iter_c3.txt 2>&1
timeout 300 python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 >> gpurun_out/iter_c3.txt 2>&1
