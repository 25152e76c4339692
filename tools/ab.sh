# A/B timing of two library builds on the same box: ab/libdvc_A.so vs ab/libdvc_B.so (built with
# `python paper_2601_20564_b200/build.py --experiments ab/libdvc_X.so`), alternating A B A B so clock
# drift cancels.  Usage (on the GPU box): bash tools/ab.sh [rounds]
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${1:-2}); do
  for v in A B; do
    printf "%s  " $v
    DVC_LIB=ab/libdvc_$v.so timeout 300 python tools/step_time.py ${ARGS} 2>&1 | tail -1
  done
done
