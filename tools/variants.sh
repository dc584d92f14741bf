#!/bin/bash
# A/B tuning runs on the GPU box: bench the in-tree library and each variant
# build (python -m paper_2603_12185_b200.build --variant TAG -D ...), interleaved.
#   tools/variants.sh OUT ROUNDS TAG... [-- bench args]
OUT=$1; shift; ROUNDS=$1; shift
TAGS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do TAGS+=("$1"); shift; done; [ "$1" == "--" ] && shift
mkdir -p gpurun_out
: > gpurun_out/$OUT
for r in $(seq $ROUNDS); do
  for t in base "${TAGS[@]}"; do
    if [ $t == base ]; then L=""; else L=paper_2603_12185_b200/_build_$t/libcomfree_$t.so; fi
    us=$(COMFREE_LIB=$L timeout 300 python bench.py --steps 200 --cpu-seconds 0.1 --e2e-steps 1 "$@" 2>/dev/null | \
      python tools/bench_line.py)
    echo "$t $us" | tee -a gpurun_out/$OUT
  done
done
