# A/B(/C) of engine builds on one box: LIBS="A:path B:path ..." bash tools/ab.sh [configs]
# (or bash tools/ab.sh LIB_A LIB_B [configs])
if [ -z "${LIBS:-}" ]; then LIBS="A:$1 B:$2"; shift 2; fi
CFGS=${@:-C1 C2 C3 C4}
for rep in 1 2; do
  for vl in $LIBS; do
    v=${vl%%:*}; lib=${vl#*:}
    for c in $CFGS; do
      CKB200_LIB=$lib python bench.py --config $c --blocks '' --no-cpu-baseline --no-e2e --no-committee \
        --no-deform --no-tc --tc-train '' --steps 20 --warmup 5 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', '$c', round(d['value']), 'eval', round(d.get('eval', {}).get('value', 0)))"
    done
  done
done
