cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_graph.txt
: > $O
echo "== C3 repeat, graph on (HMGP_TIMING)" >> $O
HMGP_TIMING=1 timeout 900 python scripts/probe_repeat.py 512 5 >> $O 2>&1
echo "== C3 repeat, graph off" >> $O
HMGP_GRAPH=0 timeout 900 python scripts/probe_repeat.py 512 3 >> $O 2>&1
echo "== C4 batches" >> $O
for T in 8 16; do
  HMGP_BATCH_THREADS=$T timeout 900 python scripts/probe_batch2.py 256 64 1e-7 16 64 >> $O 2>&1
done
HMGP_GRAPH=0 HMGP_BATCH_THREADS=8 timeout 900 python scripts/probe_batch2.py 256 64 1e-7 16 32 >> $O 2>&1
echo "== C3 batch 5 + 5" >> $O
HMGP_BATCH_KEEP=1 HMGP_BATCH_THREADS=4 timeout 1200 python scripts/probe_batch2.py 512 128 1e-6 5 5 >> $O 2>&1
cat $O
