# one gpurun call of the round's measure loop
set -x
R=${ROUND_TAG:-r02c}
timeout 600 python -m pytest tests/test_gpu_gen.py -x -q > gpurun_out/${R}_gputest_gen.log 2>&1; echo gen=$?
tail -3 gpurun_out/${R}_gputest_gen.log
for nw in 1 2; do timeout 600 python tools/strong_probe.py --nw $nw > gpurun_out/${R}_strong_nw$nw.txt 2>&1; done
cat gpurun_out/${R}_strong_nw*.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/${R}_gputest.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err; echo bench=$?
cat gpurun_out/${R}_bench_c5.json
tail -3 gpurun_out/${R}_bench_c5.err
