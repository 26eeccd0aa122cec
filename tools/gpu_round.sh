set -x
R=${ROUND_TAG:-r02s}
timeout 900 python bench.py --workload c4 --steps 3 > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
cut -c1-400 gpurun_out/${R}_bench_c4.json; tail -2 gpurun_out/${R}_bench_c4.err
timeout 900 python -m pytest -x -q tests/test_gpu_summary.py tests/test_gpu_parity.py -k "config4 or golden" > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/${R}_gputest.log
