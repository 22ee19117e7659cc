cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_graph3.txt
: > $O
for T in 8 14; do
  HMGP_BATCH_KEEP=1 HMGP_BATCH_THREADS=$T timeout 900 python scripts/probe_batch2.py 256 64 1e-7 16 96 2>&1 | grep -v "host enqueue" >> $O
done
cat $O
