# A/B of product-library builds (tools/ab_libs/lib*.so from tools/yee2_variants.sh):
# LIBS="default npt2" bash tools/yee_lib_ab.sh
mkdir -p gpurun_out/yee_lib
for cfg in ${CFGS:-yee256 yee256_f32}; do
  for rep in 1 2 3; do
    for l in ${LIBS:-default npt2}; do
      tag=${cfg}_${l}_${rep}
      if [ "$l" = default ]; then unset SFEEC_B200_LIB; else export SFEEC_B200_LIB=tools/ab_libs/lib$l.so; fi
      timeout 300 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/yee_lib/$tag.json 2> gpurun_out/yee_lib/$tag.err
      python3 -c "
import json;d=json.load(open('gpurun_out/yee_lib/$tag.json'));r=d['roofline']
print('$cfg $l', round(d['ms_per_step'],4), '%.3e'%d['value'], 'kernel_ms', round(r['kernel_avg_ms'],4), 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
unset SFEEC_B200_LIB
