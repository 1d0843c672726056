mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputests_r2i.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gputests_r2i.log
timeout 600 python bench.py --config yee256 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/yee20.json 2>/dev/null
timeout 600 python bench.py --config yee256 --no-cpu-baseline > gpurun_out/yee1000.json 2>/dev/null
timeout 600 python bench.py --config tet16 --steps 2000 --no-cpu-baseline > gpurun_out/tet16.json 2>/dev/null
for f in yee20 yee1000 tet16; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['roofline'].get('frac'), d['clocks']['sm_mhz'])"; done
