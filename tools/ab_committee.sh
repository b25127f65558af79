for rep in 1 2; do for L in B F; do
CKB200_LIB=ab/lib$L.so python bench.py --steps 10 --warmup 3 --blocks '' --no-cpu-baseline --no-e2e --no-deform --no-tc --tc-train '' 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value']), 'committee', round(d['committee']['value']), d['committee'].get('config', d['committee'].get('workload','')))"
done; done
