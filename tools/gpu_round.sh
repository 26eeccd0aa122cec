set -x
R=${ROUND_TAG:-r02w}
OTFGPU_LIB_OVERRIDE=$PWD/build/q4only/libotfgpu.so timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_summary.py -k "golden or config5_full or config3" > gpurun_out/${R}_parity.log 2>&1; echo parity=$?
tail -1 gpurun_out/${R}_parity.log
for rep in 1 2 3; do
for v in "" build/q4only/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done
done > gpurun_out/${R}_ab.txt 2>&1
unset OTFGPU_LIB_OVERRIDE
grep "^==" gpurun_out/${R}_ab.txt | cut -c1-150
