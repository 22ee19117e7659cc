cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_graph2.txt
: > $O
echo "== C4 T=4 5+8 graph timing" >> $O
HMGP_TIMING=1 HMGP_BATCH_KEEP=1 HMGP_BATCH_THREADS=4 timeout 600 python scripts/probe_batch2.py 256 64 1e-7 5 8 2>&1 | grep -v "host enqueue" >> $O
echo "== matvec tests" >> $O
timeout 600 python -m pytest tests/test_matvec_gpu.py -x -q 2>&1 | tail -15 >> $O
echo "== trace warm batch C4 T=4" >> $O
HMGP_BATCH_KEEP=1 HMGP_BATCH_THREADS=4 timeout 900 python scripts/trace_batch2.py 256 64 1e-7 5 8 >> $O 2>&1
cat $O
