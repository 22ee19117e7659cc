# A/B: descriptor ring read in place (zero-copy, default) vs per-launch H2D copies
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_desc.txt
: > $O
for mode in zc copy; do
  if [ $mode = copy ]; then export HMGP_DESC_COPY=1; else unset HMGP_DESC_COPY; fi
  echo "== mode=$mode" >> $O
  # warm + timed single C3
  timeout 600 python scripts/probe_repeat.py 512 3 >> $O 2>&1
  # C4-shaped batch: 16 theta, 8 workers
  HMGP_BATCH_THREADS=8 timeout 600 python scripts/probe_batch.py 256 64 1e-7 16 >> $O 2>&1
  HMGP_BATCH_THREADS=16 timeout 600 python scripts/probe_batch.py 256 64 1e-7 32 >> $O 2>&1
  # C3 batch of 5
  HMGP_BATCH_THREADS=4 timeout 900 python scripts/probe_batch.py 512 128 1e-6 5 >> $O 2>&1
done
cat $O
