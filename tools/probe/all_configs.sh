# device / e2e ms per clip for every BASELINE config (bench.py --config)
for c in C1 C2 C3 C4 C5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phases_ms']
print('$c', 'device %.2f ms' % d['ms_per_step'], 'e2e %.2f ms' % d['e2e']['ms_per_step'], 'fps %.0f / %.0f' % (d['value'], d['e2e']['value']), 'runs', d['config']['runs'], 'passes', d['config']['dp_passes'], 'scan %.2f' % p['scan'], 'fallbacks', p['scan_fallbacks'])"
done
