for v in 1 9 10; do
  SFEEC_SELL_VARIANT=$v timeout 600 python bench.py --config p2_64 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/sell_$v.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/sell_$v.json'));print('variant $v',round(d['ms_per_step'],3),{k:(round(v['avg_ms'],3),v.get('gbs') and round(v['gbs'])) for k,v in d['roofline'].get('per_kernel',{}).items()}, d['clocks']['sm_mhz'])"
done
