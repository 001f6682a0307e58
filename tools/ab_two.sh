#!/bin/bash
# A/B two library builds on the same box at base clocks: tools/ab_two.sh <libA> <libB> <layout> [variants]
A=$1; B=$2; L=${3:-g120p8}; V=${4:-cta2}
for lib in $A $B $A $B; do
  echo "== $lib $L"
  LLEP_LIB=$lib bash tools/ab_ncu.sh $L $V 1 | awk '{k=$3" "$4; s[k]+=$6; n[k]++; t[k]+=$8} END {for (k in s) printf "%s mean_ns %.0f tensor%% %.2f\n", k, s[k]/n[k], t[k]/n[k]}'
done
