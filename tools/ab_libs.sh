#!/bin/bash
# Same-box A/B of libpec.so builds (measurement tool): put variants at ab/libpec_<name>.so
# (git-ignored, they travel with the gpurun snapshot), then
#   gpurun -- 'bash tools/ab_libs.sh "orig lop3" "--engine crc"'
# runs bench.py (no CPU/stall/e2e legs) for each variant, alternating, three rounds, prints
# "<name> <round> ms_per_step roofline.frac avg_launch_ms", and restores the in-tree library.
set -u
variants=${1:?variant names}
args=${2:-}
mkdir -p gpurun_out
cp paper_2408_04307_b200/_lib/libpec.so ab/libpec_intree.so
for r in 1 2 3; do for v in $variants; do
  cp ab/libpec_$v.so paper_2408_04307_b200/_lib/libpec.so
  timeout 300 python bench.py $args --no-cpu --no-stall --no-e2e --steps 10 --warmup 3 \
    > gpurun_out/ab_${v}_${r}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_${v}_${r}.json')); r=d['roofline']; print('$v', $r, d['ms_per_step'], r['frac'], r['avg_launch_ms'])"
done; done
cp ab/libpec_intree.so paper_2408_04307_b200/_lib/libpec.so
