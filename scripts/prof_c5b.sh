# C5-shaped 3-D probes without stats serialisation (wall per L(θ))
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
for n in 262144 524288; do
  timeout 1200 python scripts/probe_3d.py $n >> gpurun_out/c5b_probe.txt 2>&1
  echo "n=$n rc=$?" >> gpurun_out/c5b_probe.txt
done
