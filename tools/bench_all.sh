# all configs on one B200 (round 2): JSON lines into gpurun_out/bench_all/,
# then the launch list and one ncu --set full capture of the lattice kernels
mkdir -p gpurun_out/bench_all
B=gpurun_out/bench_all
timeout 900 python bench.py > $B/tet256.json 2> $B/tet256.err
timeout 900 python bench.py --impl reference > $B/ref_tet256.json 2> $B/ref_tet256.err
timeout 900 python bench.py --config tet128 --steps 500 > $B/tet128.json 2> $B/tet128.err
timeout 600 python bench.py --config tet16 --steps 2000 > $B/tet16.json 2> $B/tet16.err
timeout 600 python bench.py --config yee256 > $B/yee256.json 2> $B/yee256.err
timeout 600 python bench.py --config yee256_f32 > $B/yee256_f32.json 2> $B/yee256_f32.err
timeout 1500 python bench.py --config p2_64 --steps 200 > $B/p2_64.json 2> $B/p2_64.err
for f in $B/*.json; do python3 -c "
import json,sys;d=json.load(open('$f'));r=d.get('roofline',{});print('$f'.split('/')[-1], '%.3e'%d['value'] if d.get('value') else None, round(d.get('ms_per_step',0) or 0,4), r.get('frac') and round(r['frac'],3), r.get('algorithmic_frac') and round(r['algorithmic_frac'],3), d.get('e2e',{}).get('value') and '%.3e'%d['e2e']['value'], d.get('cpu_baseline',{}).get('value') and '%.3e'%d['cpu_baseline']['value'], d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))"; done
if [ -n "$NCU" ]; then
  python tools/profile_kq.py tet256 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_tet256.csv python tools/profile_kq.py tet256 > gpurun_out/ncu_l.log 2>&1
  python tools/profile_kq.py tet256 > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_lat_" -c 4 \
      -o gpurun_out/lat_tet256_r2 python tools/profile_kq.py tet256 > gpurun_out/ncu.log 2>&1
  echo "ncu rc=$?"
  python tools/profile_kq.py p2_64 > gpurun_out/prof_plain3.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_p2_64.csv python tools/profile_kq.py p2_64 > gpurun_out/ncu_l2.log 2>&1
fi
