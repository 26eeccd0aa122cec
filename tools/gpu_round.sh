# the round's final evidence set (profiles/${ROUND_TAG}_*)
set -x
R=${ROUND_TAG:-r02k}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/${R}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err; echo bench=$?
timeout 900 python bench.py --workload c4 --steps 3 > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo c4=$?
timeout 900 python bench.py --workload c5t --steps 3 > gpurun_out/${R}_bench_c5t.json 2> gpurun_out/${R}_bench_c5t.err; echo c5t=$?
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err; echo ref=$?
timeout 600 python tools/strong_probe.py > gpurun_out/${R}_strong.txt 2>&1; echo strong=$?
timeout 300 python tools/e2e_breakdown.py > gpurun_out/${R}_e2e_breakdown.txt 2>&1
for tool in ${SANITIZE_TOOLS:-}; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/${R}_sanitize_$tool.txt 2>&1; echo $tool=$?
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:windowed -c 1 -o gpurun_out/${R}_windowed_c5 python tools/prof_run.py c5 > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_windowed_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/${R}_sass.csv 2>/dev/null
ncu -i gpurun_out/${R}_windowed_c5.ncu-rep --page raw --csv > gpurun_out/${R}_raw.csv 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# A/B of the final library against build/prev, when present
[ -n "${AB:-}" ] && [ -f build/prev/libotfgpu.so ] && DIAG=1 bash tools/ab.sh c5fw 2 gpurun_out/${R}_ab.txt
