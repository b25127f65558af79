# A/B of two builds of the engine on one box: bash tools/ab.sh LIB_A LIB_B [configs]
A=$1; B=$2; shift 2
CFGS=${@:-C1 C2 C3 C4}
for rep in 1 2; do
  for v in A B; do
    lib=$A; [ $v = B ] && lib=$B
    for c in $CFGS; do
      CKB200_LIB=$lib python bench.py --config $c --blocks '' --no-cpu-baseline --no-e2e --no-committee \
        --no-deform --no-tc --tc-train '' --steps 20 --warmup 5 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', '$c', round(d['value']))"
    done
  done
done
