cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32

O=gpurun_out/exp_batch_trace.txt
: > $O
HMGP_BATCH_THREADS=1 timeout 900 python scripts/trace_batch.py 256 64 1e-7 4 >> $O 2>&1
HMGP_BATCH_THREADS=8 timeout 900 python scripts/trace_batch.py 256 64 1e-7 9 >> $O 2>&1
cat $O
