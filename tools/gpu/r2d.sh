set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lattice.py -x -q > gpurun_out/lat_tests2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lat_tests2.log
python tools/profile_kq.py tet256 > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_lat_" -c 4 -o gpurun_out/lat_tet256 python tools/profile_kq.py tet256 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
