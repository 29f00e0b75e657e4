#!/bin/bash
# A/B timing of alternative builds of libhgf.so on one box: bench.py (C4 by default) with the in-tree library,
# then with each LIB argument copied over it, then the in-tree library again (drift check).
# usage: bash tools/ab_libs.sh paper_1803_00005_b200/libhgf_x.so ...   (extra bench args in $BENCH_ARGS)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
P=paper_1803_00005_b200
cp $P/libhgf.so /tmp/libhgf_base.so
run() {
  python bench.py --steps 10 $BENCH_ARGS 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1',round(d['ms_per_step'],3),{k:round(v,2) for k,v in d['stage_ms_per_step'].items() if v})"
}
run base
for lib in "$@"; do
  case "$lib" in *.gz) gunzip -c "$lib" > $P/libhgf.so ;; *) cp "$lib" $P/libhgf.so ;; esac
  run "$(basename "$lib")"
done
cp /tmp/libhgf_base.so $P/libhgf.so
run base2
