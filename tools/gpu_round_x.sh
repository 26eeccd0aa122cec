set -x
timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_summary.py -k "golden or config5_full or config4_largest or stratified or run_to_run" > gpurun_out/r02zs_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/r02zs_parity.log
for rep in 1 2 3; do
  echo "== intree rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
  echo "== prev rep $rep $(OTFGPU_LIB_OVERRIDE=$PWD/build/prev/libotfgpu.so timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done > gpurun_out/r02zs_ab.txt 2>&1
for v in "" build/prev/; do
  echo "== c5t $v $(OTFGPU_LIB_OVERRIDE=${v:+$PWD/${v}libotfgpu.so} timeout 600 python bench.py --workload c5t --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-160)"
done >> gpurun_out/r02zs_ab.txt 2>&1
grep "^==" gpurun_out/r02zs_ab.txt | cut -c1-150
