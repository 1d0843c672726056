set -x
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi; df -h /tmp /dev/shm) > gpurun_out/box.txt 2>&1
timeout 900 python bench.py --config tet256 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/tet256.json 2> gpurun_out/tet256.err
echo rc=$?
