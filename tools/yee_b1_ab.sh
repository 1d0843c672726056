# A/B of the two-step Yee sweep's one-barrier form (SFEEC_YEE_B1=2, default) vs two barriers (1)
mkdir -p gpurun_out/yee_b1
for cfg in ${CFGS:-yee256 yee256_f32}; do
  for rep in 1 2 3; do
    for v in 1 2; do
      SFEEC_YEE_B1=$v timeout 300 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/yee_b1/${cfg}_${v}_${rep}.json 2> gpurun_out/yee_b1/${cfg}_${v}_$rep.err
      python3 -c "
import json;d=json.load(open('gpurun_out/yee_b1/${cfg}_${v}_${rep}.json'));r=d['roofline']
print('$cfg B1=$v', round(d['ms_per_step'],4), '%.3e'%d['value'], 'kernel_ms', round(r['kernel_avg_ms'],4), 'frac', round(r['frac'],3), 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
