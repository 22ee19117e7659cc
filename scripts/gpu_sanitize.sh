# compute-sanitizer on a C1-shaped L(θ): memcheck + racecheck + synccheck
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/probe_phases.py 32 64 1e-7 1.0,0.1,0.5,0.01 ldl > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|wall" gpurun_out/sanitizer_$tool.log | tail -3
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python scripts/probe_phases.py 64 64 1e-7 1.0,0.1,1.0,0.01 cholesky > gpurun_out/sanitizer_memcheck_c1.log 2>&1
echo "memcheck C1 rc=$?"; grep -E "ERROR SUMMARY|wall" gpurun_out/sanitizer_memcheck_c1.log | tail -3
