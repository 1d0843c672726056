# A/B of the L2 prefetch-size hint on the operator streams (SFEEC_L2PF=0/1/2)
mkdir -p gpurun_out/l2pf
summ() { python3 -c "
import json,sys
d=json.load(open('$1'));r=d['roofline']
print('$2', round(d['ms_per_step'],4), '%.3e'%d['value'], 'frac', round(r['frac'],3), 'step', round(r.get('step_achieved_gbs',0)), {k:(round(v['avg_ms'],3), v.get('gbs') and round(v['gbs'])) for k,v in r.get('per_kernel',{}).items()}, d['clocks']['sm_mhz'])"; }
for cfg in ${CFGS:-tet128}; do
  for rep in 1 2; do
  for v in ${VARIANTS:-"SFEEC_L2PF=0" "SFEEC_L2PF=2" "SFEEC_L2PF=1" "SFEEC_L2PF=4" "SFEEC_L2PF=6"}; do
    tag=$(echo "$cfg $v $rep" | tr ' =' '__')
    env $v timeout 900 python bench.py --config $cfg --steps ${STEPS:-300} --warmup 5 --no-cpu-baseline > gpurun_out/l2pf/$tag.json 2> gpurun_out/l2pf/$tag.err
    summ gpurun_out/l2pf/$tag.json "$cfg $v"
  done
  done
done
