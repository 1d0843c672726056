set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gputests_full.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/gputests_full.log
