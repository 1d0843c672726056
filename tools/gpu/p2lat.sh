# table-lattice tests, the config-4 full-size parity test, then config 4
# (p2_64) on the lattice vs the sliced step
mkdir -p gpurun_out/p2lat
timeout 1000 python -m pytest tests/test_gpu_table_lattice.py tests/test_gpu_p2.py -x -q 2>&1 | tail -3
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -k config4 2>&1 | tail -3
for lay in ${LAYOUTS:-device sell}; do
  SFEEC_P2_LAYOUT=$lay timeout 1500 python bench.py --config p2_64 --steps ${STEPS:-200} --warmup 3 > gpurun_out/p2lat/p2_64_$lay.json 2> gpurun_out/p2lat/p2_64_$lay.err
  tail -3 gpurun_out/p2lat/p2_64_$lay.err
  python -c "
import json; d=json.load(open('gpurun_out/p2lat/p2_64_$lay.json')); r=d['roofline']['per_kernel']
print('$lay', round(d['ms_per_step'],4), '%.3e'%d['value'], {k: (round(x['avg_ms'],4), round(x.get('gbs',0))) for k,x in r.items()}, d['clocks']['sm_mhz'], d['config'].get('host_setup_s'), 'e2e %.3e' % d['e2e']['value'])"
done
