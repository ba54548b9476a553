for t in 0 256 192 128 0 256 192 128; do
  RAMLT_MIX_COOP_THREADS=$t timeout 300 python bench.py --workload c2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads=$t', round(d['value']/1e9,2), 'G steps/s', 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,2))"
done
