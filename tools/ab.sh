# A/B timing of the in-tree library against build/prev (tools/probe.py; not part of the product)
# usage: [DIAG=1] bash tools/ab.sh <probe-mode> <reps> [out]
MODE=${1:-c5fw}; REPS=${2:-2}; OUT=${3:-gpurun_out/ab.txt}
for rep in $(seq 1 $REPS); do
for v in intree prev; do
  if [ $v = intree ]; then unset OTFGPU_LIB_OVERRIDE; else export OTFGPU_LIB_OVERRIDE=$PWD/build/prev/libotfgpu.so; fi
  r=$(OTF_DIAG=${DIAG:-} timeout 300 python tools/probe.py $MODE 2>&1)
  echo "== $v rep $rep $(echo "$r" | tail -1)"
  echo "$r" | head -n -1 | cut -c1-400
done
done > $OUT 2>&1
unset OTFGPU_LIB_OVERRIDE
grep "^==" $OUT | sed 's/"requests".*"req_per_s"/ req_per_s/'
