mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -q > gpurun_out/slab_ov.log 2>&1; echo "overlap rc=$?"; tail -2 gpurun_out/slab_ov.log
SFEEC_PART_OVERLAP=0 timeout 900 python -m pytest tests/test_gpu_slabs.py -q > gpurun_out/slab_noov.log 2>&1; echo "serial rc=$?"; tail -2 gpurun_out/slab_noov.log
