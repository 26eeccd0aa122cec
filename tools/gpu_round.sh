set -x
R=${ROUND_TAG:-r02v}
timeout 900 python bench.py --workload c4 --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
cut -c1-300 gpurun_out/${R}_bench_c4.json
timeout 900 python -m pytest -x -q tests/test_gpu_summary.py tests/test_gpu_parity.py -k "config4 or golden" > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -1 gpurun_out/${R}_gputest.log
