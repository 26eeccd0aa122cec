set -x
R=${ROUND_TAG:-r02x}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo gputest=$?
tail -2 gpurun_out/${R}_gputest.log
OTF_DIAG=1 timeout 600 python tools/probe.py c5fw c5tw c4T10k > gpurun_out/${R}_probe.txt 2>&1; echo probe=$?
cat gpurun_out/${R}_probe.txt | cut -c1-400
