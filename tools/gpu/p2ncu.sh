mkdir -p gpurun_out/p2ncu
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_tl_" -c 4 \
    -o gpurun_out/p2ncu/tl_p2_64 python tools/profile_kq.py p2_64 > gpurun_out/p2ncu/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/p2ncu/tl_p2_64.ncu-rep --page raw --csv > gpurun_out/p2ncu/tl_p2_64_raw.csv 2>/dev/null
