#!/bin/bash
# Same-box A/B of prebuilt libraries (ab/lib_<V>.so): the in-tree library is
# swapped before every run; device lines of the configs in $CFGS (default
# "cfg4 cfg2") for the variants in $VARS (default "A B"), alternating, two
# rounds.  Profiling only.
mkdir -p gpurun_out
LIB=paper_1610_01108_b200/libamun_b200.so
cp $LIB /tmp/ab_orig.so
for r in 1 2; do for v in ${VARS:-A B}; do
  cp ab/lib_$v.so $LIB
  for c in ${CFGS:-cfg4 cfg2}; do
    timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_${c}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_${c}_$r.json').read().strip().splitlines()[-1]);print('$v $c $r', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done; done
cp /tmp/ab_orig.so $LIB
