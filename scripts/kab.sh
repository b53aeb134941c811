mkdir -p gpurun_out
for k in fine lanes tile; do
python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-trace --no-render --kernel $k > gpurun_out/k_$k.json 2>gpurun_out/k_$k.err
python -c "import json; d=json.load(open('gpurun_out/k_$k.json')); r=d['roofline']; print('$k', 'kernel ms', r['launch_ms'], 'step', round(d['ms_per_step'],3), 'Gq/s', round(d['value']/1e9,2), 'frac', round(r['frac'],4), d['counters'])"
done
