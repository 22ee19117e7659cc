cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/exp_graph4.txt
: > $O
echo "== C4 T=16 one-stream workers: 16 (cold) + 48 + 64" >> $O
timeout 600 python scripts/probe_batch3.py 256 64 1e-7 16 48 64 >> $O 2>&1
echo "== C4 T=16 workers with sections" >> $O
HMGP_BATCH_SECTIONS=1 timeout 600 python scripts/probe_batch3.py 256 64 1e-7 16 48 64 >> $O 2>&1
echo "== C3 sections workers: 5 + 6 + 6" >> $O
HMGP_BATCH_SECTIONS=1 timeout 900 python scripts/probe_batch3.py 512 128 1e-6 5 6 6 >> $O 2>&1
echo "== C3 one-stream workers: 5 + 6 + 6" >> $O
timeout 900 python scripts/probe_batch3.py 512 128 1e-6 5 6 6 >> $O 2>&1
cat $O
