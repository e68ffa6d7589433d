#!/bin/bash
# A/B of dropout-mask variant builds (dev): bash scripts/ab_mask.sh tag ...  ("base" = libub.so)
for T in "$@"; do
  if [ "$T" = "base" ]; then LIBF=paper_2208_08124_b200/libub.so; else LIBF=paper_2208_08124_b200/libub_$T.so; fi
  echo -n "$T: "; UB_LIB=$LIBF timeout -k 5 60 python scripts/probe_mask.py
done
