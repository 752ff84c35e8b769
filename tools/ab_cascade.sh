#!/bin/bash
# A/B the cascade across library variants built by `make variant` (csrc/build/var_*).
# usage: tools/ab_cascade.sh [m n] ; prints one line per variant per round.
M=${1:-2000}; N=${2:-20000}
cd "$(dirname "$0")/.."
for round in 1 2; do
  for v in default paper_1502_03543_b200/csrc/build/var_*; do
    if [ "$v" = default ]; then lib=paper_1502_03543_b200/libpdas_b200.so; name=default;
    else lib=$v/libpdas_b200.so; name=$(basename $v); fi
    r=$(PDAS_B200_LIB=$lib timeout 120 python tools/cascade_time.py --m $M --n $N --reps 2 2>&1 | tail -1)
    echo "$name: $r"
  done
done
