# GPU validation pass: tests, smoke, bench; logs under gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-s}
python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu_$T.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$T.log
python __graft_entry__.py smoke >> gpurun_out/pytest_gpu_$T.log 2>&1
tail -4 gpurun_out/pytest_gpu_$T.log
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench_rc=$?
tail -3 gpurun_out/bench_$T.err
head -c 1500 gpurun_out/bench_$T.json
