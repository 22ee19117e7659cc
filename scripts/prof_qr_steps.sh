mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
HMGP_STATS=1 timeout 300 python scripts/bench_trunc.py 2 256,256,0,96 > gpurun_out/qr_96.txt 2>&1
HMGP_STATS=1 timeout 300 python scripts/bench_trunc.py 2 1024,1024,0,96 > gpurun_out/qr_1024.txt 2>&1
