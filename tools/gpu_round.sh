set -x
R=${ROUND_TAG:-r02q}
for rep in 1 2 3; do
for v in "" build/noprefix/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== $name rep $rep $(timeout 300 python tools/probe.py c5fw 2>&1 | tail -1)"
done
done > gpurun_out/${R}_ab.txt 2>&1
for v in "" build/noprefix/; do
  if [ -z "$v" ]; then unset OTFGPU_LIB_OVERRIDE; name=intree; else export OTFGPU_LIB_OVERRIDE=$PWD/${v}libotfgpu.so; name=$(basename $v); fi
  echo "== c4 $name $(timeout 600 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200)"
done >> gpurun_out/${R}_ab.txt 2>&1
unset OTFGPU_LIB_OVERRIDE
grep "^==" gpurun_out/${R}_ab.txt | cut -c1-150
