set -x
R=${ROUND_TAG:-r02n}
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_summary.py -k "golden or config5_full or config4_largest or list_overflow or config3" > gpurun_out/${R}_parity.log 2>&1; echo parity=$?
tail -2 gpurun_out/${R}_parity.log
for rep in 1 2 3; do
for v in "" build/noprefix/ build/q64/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done
done > gpurun_out/${R}_ab.txt 2>&1
for v in "" build/noprefix/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== c5t $name $(timeout 600 python bench.py --workload c5t --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200)"
done >> gpurun_out/${R}_ab.txt 2>&1
unset OTFGPU_LIB_OVERRIDE
grep "^==" gpurun_out/${R}_ab.txt | cut -c1-150
