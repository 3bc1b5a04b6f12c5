#!/bin/bash
# A/B device-time comparison of two library builds on the same box: tools/ab.sh libA libB case [reps] [rounds]
A=$(realpath $1); B=$(realpath $2); C=$3; R=${4:-5}; N=${5:-2}
for i in $(seq $N); do
  for L in $A $B; do
    echo -n "$(basename $L) "; UNSO_LIB=$L timeout 300 python tools/stage_profile.py $C $R 2>&1 | tail -1 | cut -c1-330
  done
done
