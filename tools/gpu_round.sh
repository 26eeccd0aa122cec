set -x
R=${ROUND_TAG:-r02k}
OTFGPU_LIB_OVERRIDE=$PWD/build/qsort/libotfgpu.so timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_summary.py -k "golden or config5_full or config5_point or config3 or config2" > gpurun_out/${R}_parity_qsort.log 2>&1; echo parity_qsort=$?
tail -2 gpurun_out/${R}_parity_qsort.log
for rep in 1 2 3; do
for v in "" build/qsort/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done
done > gpurun_out/${R}_ab.txt 2>&1
cat gpurun_out/${R}_ab.txt | cut -c1-130
