# A/B the two-step sweep builds of tools/ab_libs (tools/yee2_variants.sh) against the in-tree library
for lib in "" $(ls tools/ab_libs/*.so 2>/dev/null); do for cfg in yee256 yee256_f32; do
  SFEEC_B200_LIB=$lib timeout 600 python bench.py --config $cfg --steps 1000 --no-cpu-baseline > gpurun_out/ab2.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/ab2.json'));r=d['roofline'];print('${lib:-in-tree}', '$cfg', round(d['ms_per_step'],4), round(r['kernel_avg_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
