for cfg in tet128 p2_32; do for v in 9 11 12 13; do
  SFEEC_SELL_VARIANT=$v timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/sell_${cfg}_$v.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/sell_${cfg}_$v.json'));print('$cfg variant $v',round(d['ms_per_step'],3),{k:(round(v['avg_ms'],3),v.get('gbs') and round(v['gbs'])) for k,v in d['roofline'].get('per_kernel',{}).items() if k=='K-Q'}, d['clocks']['sm_mhz'])"
done; done
