# A/B timing of two library builds on the same box: ab/libdvc_A.so vs ab/libdvc_B.so, alternating
# A B A B so clock drift cancels.  Usage (on the GPU box): bash tools/ab.sh [rounds]
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${1:-2}); do
  for v in A B; do
    echo "== $v"
    DVC_LIB=ab/libdvc_$v.so timeout 120 python tools/conv_breakdown.py 2>/dev/null | head -1
    DVC_LIB=ab/libdvc_$v.so timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps', round(d['value'],1))"
  done
done
