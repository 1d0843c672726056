# A/B of programmatic dependent launch (SFEEC_PDL=0/1)
mkdir -p gpurun_out/pdl
for cfg in ${CFGS:-tet16 tet128 yee256}; do
  st=300; [ $cfg = tet16 ] && st=2000
  for rep in 1 2; do
    for v in 0 1; do
      SFEEC_PDL=$v timeout 600 python bench.py --config $cfg --steps $st --no-cpu-baseline > gpurun_out/pdl/${cfg}_${v}_${rep}.json 2> gpurun_out/pdl/${cfg}_${v}_${rep}.err
      python3 -c "
import json;d=json.load(open('gpurun_out/pdl/${cfg}_${v}_${rep}.json'))
print('$cfg PDL=$v', round(d['ms_per_step'],5), '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
