set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
HMGP_DAG_DIAG=1 timeout 300 python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 > gpurun_out/c3_dag.txt 2>&1
echo dag_rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 1 --warmup 0 --no-extras --no-cpu-baseline > gpurun_out/c3_ncu_bench.log 2>&1
echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_truncate_cluster -s 300 -c 2 -o gpurun_out/c3_trunc_cluster python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 > gpurun_out/c3_ncu_full.log 2>&1
echo ncufull_rc=$?
