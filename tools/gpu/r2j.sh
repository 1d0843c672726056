mkdir -p gpurun_out
python tools/profile_kq.py tet128 > gpurun_out/p128.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_lat_" -c 4 -o gpurun_out/lat_tet128_r2 python tools/profile_kq.py tet128 > gpurun_out/ncu128.log 2>&1
echo "ncu rc=$?"
