cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/exp_solve.txt
: > $O
for G in 148 96 64 32 16; do
  echo "== grid $G" >> $O
  HMGP_SOLVE_GRID=$G HMGP_SOLVE_STATS=1 timeout 300 python scripts/probe_hbm.py 512 solve 2>&1 | grep -E "solve|matvec" >> $O
done
cat $O
