# A/B/n timing of build/<variant>/libotfgpu.so libraries (tools/probe.py; not part of the product)
# usage: [DIAG=1] bash tools/abn.sh <probe-mode> <reps> <out> variant...
MODE=$1; REPS=$2; OUT=$3; shift 3
for rep in $(seq 1 $REPS); do
for v in "$@"; do
  export OTFGPU_LIB_OVERRIDE=$PWD/build/$v/libotfgpu.so
  r=$(OTF_DIAG=${DIAG:-} timeout 300 python tools/probe.py $MODE 2>&1)
  echo "== $v rep $rep $(echo "$r" | tail -1)"
  echo "$r" | head -n -1 | cut -c1-400
done
done > $OUT 2>&1
unset OTFGPU_LIB_OVERRIDE
grep "^==" $OUT | sed 's/"requests".*"req_per_s"/ req_per_s/'
