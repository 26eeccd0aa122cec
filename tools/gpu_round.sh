set -x
R=${ROUND_TAG:-r02y}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/${R}_gputest.log
timeout 600 python tools/c4_probe.py --classes 3000,10000 > gpurun_out/${R}_c4_probe.txt 2>&1; echo c4probe=$?
timeout 900 python bench.py --workload c4 --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
cut -c1-300 gpurun_out/${R}_bench_c4.json
