# Round-2 ncu evidence (each only after the same command ran clean without ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
# (1) HBM kernels: matvec + solve, full sets -> DRAM traffic per launch
timeout 600 python scripts/probe_hbm.py 512 solve > gpurun_out/r2_hbm_plain.txt 2>&1; echo "hbm plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_mv_|k_solve_sweep' -c 12 \
  -o gpurun_out/r2_hbm_kernels python scripts/probe_hbm.py 512 solve > gpurun_out/r2_hbm_ncu.log 2>&1; echo "hbm ncu rc=$?"
ncu -i gpurun_out/r2_hbm_kernels.ncu-rep --page raw --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed \
  > gpurun_out/r2_hbm_kernels_raw.csv 2>/dev/null; echo "hbm csv rc=$?"
# (2) top factorization kernel, full set, two launches in the middle of a C3 L(θ)
HMGP_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_truncate_pair -s 300 -c 2 \
  -o gpurun_out/r2_c3_trunc_pair python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 > gpurun_out/r2_c3_trunc_pair.log 2>&1; echo "pair ncu rc=$?"
ncu -i gpurun_out/r2_c3_trunc_pair.ncu-rep --page raw --csv > gpurun_out/r2_c3_trunc_pair_raw.csv 2>/dev/null
HMGP_GRAPH=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_gemm$' -s 2000 -c 3 \
  -o gpurun_out/r2_c3_gemm python scripts/probe_phases.py 512 128 1e-6 1.5,0.05,1.0,0.01 > gpurun_out/r2_c3_gemm.log 2>&1; echo "gemm ncu rc=$?"
ncu -i gpurun_out/r2_c3_gemm.ncu-rep --page raw --csv > gpurun_out/r2_c3_gemm_raw.csv 2>/dev/null
# (3) launch list of the bench command (stream path, first full L(θ) only)
HMGP_GRAPH=0 timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none -c 93000 --csv \
  --log-file gpurun_out/r2_c3_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-extras --no-cpu-baseline \
  > gpurun_out/r2_c3_ncu_bench.log 2>&1; echo "launch list rc=$?"
python scripts/agg_launches.py gpurun_out/r2_c3_bench_launches.csv 20 > gpurun_out/r2_c3_bench_launch_summary.txt 2>&1
gzip -f gpurun_out/r2_c3_bench_launches.csv
cat gpurun_out/r2_hbm_plain.txt; head -c 3000 gpurun_out/r2_hbm_kernels_raw.csv; cat gpurun_out/r2_c3_bench_launch_summary.txt
