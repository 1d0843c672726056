# A/B of sliced SpMV variants (tests of every layout, then bench per variant)
# usage: bash tools/delta_ab.sh [configs...]
mkdir -p gpurun_out/delta
timeout 900 python -m pytest tests/test_gpu_delta.py -x -q > gpurun_out/delta/test.log 2>&1 || { tail -60 gpurun_out/delta/test.log; exit 1; }
python tools/delta_probe.py 128 > gpurun_out/delta/layout128.txt 2>&1
cfgs="${@:-tet128 p2_64}"
for cfg in $cfgs; do
  st=500; [ $cfg = p2_64 ] && st=60
  for v in "SFEEC_SELL_TMA=0" "SFEEC_SELL_TMA=1"; do
    env $v timeout 900 python bench.py --config $cfg --steps $st --no-cpu-baseline > gpurun_out/delta/$cfg.$v.json 2> gpurun_out/delta/$cfg.$v.err
  done
done
cat gpurun_out/delta/layout128.txt
for f in gpurun_out/delta/*.json; do python3 -c "
import json;d=json.load(open('$f'));r=d.get('roofline',{})
print('$f'.split('/')[-1], '%.4e'%d['value'], round(d['ms_per_step'],4), round(r.get('frac',0),3), {k: round(v['avg_ms'],4) for k,v in r.get('per_kernel',{}).items()})"; done
