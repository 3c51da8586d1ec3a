#!/bin/bash
# Repeatability of the headline lines (tools/gpu_repeat.sh) + compute-sanitizer memcheck on the
# copy-engine / host_io paths added in round 1's second session.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
bash tools/gpu_repeat.sh
S=gpurun_out/sanitizer2.txt; : > $S
echo "## memcheck: pytest host_io + copy-engine load modes" >> $S
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -x -k "host_io or copy_engine" >> $S 2>&1; echo "rc=$?" >> $S
echo "## synccheck: pytest host_io (ring 2) + copy-engine baselines" >> $S
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests -m gpu -q -x -k "host_io" >> $S 2>&1; echo "rc=$?" >> $S
grep -E "^##|passed|failed|SUMMARY|rc=" $S
