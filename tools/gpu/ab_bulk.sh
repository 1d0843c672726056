mkdir -p gpurun_out
SFEEC_LAT_BULK=1 timeout 600 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_slabs.py -x -q > gpurun_out/bulk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/bulk_tests.log
for v in ${VARIANTS:-0 1 2 0 1 2}; do
  SFEEC_LAT_BULK=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --config ${CFG:-tet256} > gpurun_out/abb_v$v.json 2> gpurun_out/abb_v$v.err
  python -c "
import json; d=json.load(open('gpurun_out/abb_v$v.json')); r=d['roofline']['per_kernel']
print('bulk=$v', round(d['ms_per_step'],4), {k: round(x['avg_ms'],4) for k,x in r.items()}, d['clocks']['sm_mhz'])"
done
