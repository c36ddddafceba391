#!/bin/bash
# sweep the face solver's reach multipliers on configs[1] (device march time)
for cfg in "1 4 128" "2 4 128" "2 4 192" "2 6 256" "1.5 4 160" "3 6 256"; do
  set -- $cfg
  echo "tau_mult=$1 near_reach=$2 near_cap=$3: $(AM_TAU_MULT=$1 AM_NEAR_REACH=$2 AM_NEAR_CAP=$3 python tools/profile_march.py --repeat 4 | grep cells | tail -1)"
done
