# one gpurun call of the round's measure loop
set -x
R=${ROUND_TAG:-r02f}
for v in pfresp pf_unroll1; do
  OTFGPU_LIB_OVERRIDE=$PWD/build/$v/libotfgpu.so timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "golden_parity or config5_point or config4_largest" > gpurun_out/${R}_parity_$v.log 2>&1; echo parity_$v=$?
done
for rep in 1 2 3; do
for v in build/prev/ "" build/pfresp/ build/pf_unroll1/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done
done > gpurun_out/${R}_ab.txt 2>&1
unset OTFGPU_LIB_OVERRIDE
cat gpurun_out/${R}_ab.txt | cut -c1-150
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/${R}_gputest.log
