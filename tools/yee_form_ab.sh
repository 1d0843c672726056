# A/B of two-step Yee sweep forms: VARIANTS="SFEEC_YEE_ORD=0 SFEEC_YEE_ORD=1" bash tools/yee_form_ab.sh
mkdir -p gpurun_out/yee_form
for cfg in ${CFGS:-yee256 yee256_f32}; do
  for rep in 1 2 3; do
    for v in ${VARIANTS:-"SFEEC_YEE_ORD=0" "SFEEC_YEE_ORD=1"}; do
      tag=$(echo "${cfg}_${v}_${rep}" | tr ' =' '__')
      env $v timeout 300 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/yee_form/$tag.json 2> gpurun_out/yee_form/$tag.err
      python3 -c "
import json;d=json.load(open('gpurun_out/yee_form/$tag.json'));r=d['roofline']
print('$cfg $v', round(d['ms_per_step'],4), '%.3e'%d['value'], 'kernel_ms', round(r['kernel_avg_ms'],4), 'frac', round(r['frac'],3), 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
