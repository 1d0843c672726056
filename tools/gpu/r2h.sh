set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_l2_error.py -q -s > gpurun_out/l2.log 2>&1; echo "l2 rc=$?"; tail -5 gpurun_out/l2.log
timeout 600 python bench.py --config tet128 --partitioned --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/b_part128.json 2> gpurun_out/b_part128.err; echo "part rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --dist --config tet256 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/b_dist256.json 2> gpurun_out/b_dist256.err; echo "dist rc=$?"
tail -3 gpurun_out/b_dist256.err
