set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_tetdev.py tests/test_gpu_tet.py -x -q > gpurun_out/lat_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/lat_tests.log
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b_tet256_lat.json 2> gpurun_out/b_tet256_lat.err; echo "bench rc=$?"
timeout 900 python bench.py --config tet128 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b_tet128_lat.json 2> gpurun_out/b_tet128_lat.err; echo "bench128 rc=$?"
