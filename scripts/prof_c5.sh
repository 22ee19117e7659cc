# C5-shaped 3-D probes (uniform points in [0,1]^3, theta=(1,0.08,0.5,0.005), leaf 128, eps 1e-5)
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total --format=csv
for n in 131072 262144 524288 1048576; do
  timeout 900 python scripts/probe_3d.py $n >> gpurun_out/c5_probe.txt 2>&1
  echo "n=$n rc=$?" >> gpurun_out/c5_probe.txt
done
