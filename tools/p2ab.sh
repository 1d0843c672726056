set -x
for v in "SFEEC_WIDE_CSR=0" "SFEEC_WIDE_U=2" "SFEEC_WIDE_U=4" "SFEEC_WIDE_U=8"; do
  env $v timeout 600 python bench.py --config p2_32 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python3 -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v',d['ms_per_step'],{k:(round(v['avg_ms'],4),v.get('gbs') and round(v['gbs'])) for k,v in d['roofline'].get('per_kernel',{}).items()})"
done
