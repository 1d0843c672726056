for v in 2 4; do for cfg in yee256 yee256_f32; do
  SFEEC_YEE_VARIANT=$v timeout 600 python bench.py --config $cfg --steps 1000 --no-cpu-baseline > gpurun_out/yee_${cfg}_$v.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/yee_${cfg}_$v.json'));r=d['roofline'];print('$cfg v$v', d['value'], round(d['ms_per_step'],4), round(r['kernel_avg_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
