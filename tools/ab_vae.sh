# A/B of two library builds (ab/libdvc_A.so, ab/libdvc_B.so) on the same box: headline bench + VAE decoder
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  for v in A B; do
    b=$(DVC_LIB=ab/libdvc_$v.so timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
    f=$(DVC_LIB=ab/libdvc_$v.so timeout 300 python tools/bench_f2.py --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['frames_per_s'],1))")
    echo "$v bench=$b vae=$f"
  done
done
