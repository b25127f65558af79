set -x
for c in C1 C2 C3 C4; do
python bench.py --config $c --blocks '' --no-cpu-baseline --no-e2e --no-committee --no-deform --no-tc --tc-train '' --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'], round(d['value']), d['ms_per_step'])"
done
python tools/phases.py C3 2>&1 | tail -12
