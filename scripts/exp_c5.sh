# C5-shaped 3-D probes with forced starting capacities (which bound overflows at the 2-D start?)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/exp_c5.txt
: > $O
for cfg in "256 2" "512 1"; do
  set -- $cfg
  echo "== n=262144 tcap=$1 grow=$2" >> $O
  HMGP_TIMING=1 HMGP_TCAP=$1 HMGP_GROW=$2 timeout 700 python scripts/probe_3d.py 262144 2>&1 | grep -v "^\[hmgp\] graph" | tail -4 >> $O
done
cat $O
