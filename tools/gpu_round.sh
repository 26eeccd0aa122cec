set -x
R=${ROUND_TAG:-r02j}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/${R}_gputest.log
timeout 900 python bench.py > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err; echo bench=$?
cat gpurun_out/${R}_bench_c5.json; tail -2 gpurun_out/${R}_bench_c5.err
timeout 900 python bench.py --workload c4 --steps 3 > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
timeout 900 python bench.py --workload c5t --steps 3 --no-cpu-baseline > gpurun_out/${R}_bench_c5t.json 2> gpurun_out/${R}_bench_c5t.err; echo c5t=$?
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err; echo ref=$?
timeout 900 python bench.py --scaling strong > gpurun_out/${R}_bench_strong_n1.json 2> gpurun_out/${R}_bench_strong_n1.err; echo strong=$?
