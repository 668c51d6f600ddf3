# short bench run (no serving sweep, no CPU baseline) and the named legs of its JSON line
RDKV_SKIP_CPU=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-serve "$@" > gpurun_out/bq.json 2> gpurun_out/bq.err; echo rc=$?
tail -3 gpurun_out/bq.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bq.json').read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],3), d['clocks'])
print({k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})
print('decode', json.dumps(d.get('decode')))
print('ttft', json.dumps(d.get('ttft_ms')))
PY
