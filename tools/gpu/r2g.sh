set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_l2_error.py tests/test_multigpu.py tests/test_gpu_lattice.py -q -s --durations=10 > gpurun_out/slab_tests.log 2>&1; echo "tests rc=$?"
tail -40 gpurun_out/slab_tests.log
