for g in 0 1; do for cfg in tet16 tet128; do
  SFEEC_GRAPHS=$g timeout 600 python bench.py --config $cfg --steps 1000 --no-cpu-baseline > gpurun_out/g_${cfg}_$g.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/g_${cfg}_$g.json'));print('$cfg graphs=$g', '%.3e'%d['value'], round(d['ms_per_step']*1e3,2),'us/step', 'e2e %.3e'%d['e2e']['value'], d['gpu_launches'])"
done; done
