# all configs, one B200; JSON lines into gpurun_out/bench_all/
mkdir -p gpurun_out/bench_all
python bench.py > gpurun_out/bench_all/yee256.json 2> gpurun_out/bench_all/yee256.err
python bench.py --config yee256_f32 > gpurun_out/bench_all/yee256_f32.json 2> gpurun_out/bench_all/yee256_f32.err
python bench.py --config tet16 --steps 2000 > gpurun_out/bench_all/tet16.json 2> gpurun_out/bench_all/tet16.err
python bench.py --config tet128 --steps 500 > gpurun_out/bench_all/tet128.json 2> gpurun_out/bench_all/tet128.err
timeout 1200 python bench.py --config p2_64 --steps 200 > gpurun_out/bench_all/p2_64.json 2> gpurun_out/bench_all/p2_64.err
timeout 1500 python bench.py --config tet256 --steps 200 > gpurun_out/bench_all/tet256.json 2> gpurun_out/bench_all/tet256.err
python bench.py --impl reference --steps 20 > gpurun_out/bench_all/ref_yee256.json 2> gpurun_out/bench_all/ref_yee256.err
for f in gpurun_out/bench_all/*.json; do python3 -c "
import json,sys;d=json.load(open('$f'));r=d.get('roofline',{});print('$f'.split('/')[-1], '%.3e'%d['value'] if d.get('value') else None, round(d.get('ms_per_step',0) or 0,4), r.get('frac') and round(r['frac'],3), d.get('e2e',{}).get('value') and '%.3e'%d['e2e']['value'], d.get('cpu_baseline',{}).get('value') and '%.3e'%d['cpu_baseline']['value'], d.get('clocks',{}).get('reasons'))"; done
