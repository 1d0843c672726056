set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputests_full.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gputests_full.log
