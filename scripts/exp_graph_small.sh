cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_graph_small.txt
: > $O
for g in 64 128 256; do
  echo "== repeat g=$g graph on" >> $O
  HMGP_TIMING=1 timeout 300 python scripts/probe_repeat.py $g 4 >> $O 2>&1
  echo "rc=$?" >> $O
done
echo "== batch g=128" >> $O
HMGP_TIMING=1 HMGP_BATCH_THREADS=4 timeout 300 python scripts/probe_batch2.py 128 64 1e-7 8 16 >> $O 2>&1
echo "rc=$?" >> $O
cat $O
