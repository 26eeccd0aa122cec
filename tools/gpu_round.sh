# one gpurun call of the round's measure loop
set -x
R=${ROUND_TAG:-r02e}
for v in regsort regsort_pf; do
  OTFGPU_LIB_OVERRIDE=$PWD/build/$v/libotfgpu.so timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "golden_parity or config5_point or config4_largest or config2_full" > gpurun_out/${R}_parity_$v.log 2>&1; echo parity_$v=$?
  tail -2 gpurun_out/${R}_parity_$v.log
done
for rep in 1 2; do
for v in "" build/pfresp/ build/regsort/ build/regsort_pf/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep"; timeout 300 python tools/probe.py c5fw 2>&1 | tail -1
done
done > gpurun_out/${R}_ab.txt 2>&1
unset OTFGPU_LIB_OVERRIDE
cat gpurun_out/${R}_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/${R}_gputest.log
timeout 900 python bench.py --workload c5t --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c5t.json 2> gpurun_out/${R}_bench_c5t.err; echo bench_c5t=$?
timeout 600 python bench.py --workload c4 --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/${R}_sanitize_racecheck.txt 2>&1; echo racecheck=$?
tail -3 gpurun_out/${R}_sanitize_racecheck.txt
