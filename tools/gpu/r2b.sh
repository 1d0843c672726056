set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gputests.log
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/b_tet256.json 2> gpurun_out/b_tet256.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 200 --warmup 5 > gpurun_out/ref_tet256.json 2> gpurun_out/ref_tet256.err; echo "ref rc=$?"
