# A/B of the fused wavefront half-steps (wave.cu) against the 4-kernel chain
mkdir -p gpurun_out/wave
summ() { python3 -c "
import json,sys
d=json.load(open('$1'));r=d['roofline']
print('$2', round(d['ms_per_step'],4), '%.3e'%d['value'], 'frac', round(r['frac'],3), 'step', round(r.get('step_achieved_gbs',0)), {k:(round(v['avg_ms'],3), v.get('gbs') and round(v['gbs'])) for k,v in r.get('per_kernel',{}).items()}, d['clocks']['sm_mhz'])"; }
for cfg in ${CFGS:-tet128}; do
  for v in ${VARIANTS:-"SFEEC_WAVE=0" "SFEEC_WAVE=1"}; do
    tag=$(echo "$cfg $v" | tr ' =' '__')
    env $v timeout 900 python bench.py --config $cfg --steps ${STEPS:-300} --warmup 5 --no-cpu-baseline > gpurun_out/wave/$tag.json 2> gpurun_out/wave/$tag.err
    summ gpurun_out/wave/$tag.json "$cfg $v"
  done
done
