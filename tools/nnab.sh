# A/B of tracking GN iterations/s: libsgad variants in variants/ vs the tree's build
for v in "$@"; do
  echo "== $v" >> gpurun_out/r2_nnab.log
  SGAD_LIB=$( [ "$v" = tree ] && echo paper_2603_21055_b200/libsgad.so || echo variants/$v.so ) \
    timeout 200 python tools/track_bench.py 20 5 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],1), round(d['ms_per_iteration'],3))" >> gpurun_out/r2_nnab.log 2>&1
done
