#!/bin/bash
# A/B timing of variant builds (dev): for each libub_<tag>.so given, run probe_time twice.
# Usage: bash scripts/ab_libs.sh tag1 tag2 ...   (tag "base" = libub.so)
for T in "$@"; do
  if [ "$T" = "base" ]; then LIBF=paper_2208_08124_b200/libub.so; else LIBF=paper_2208_08124_b200/libub_$T.so; fi
  for i in 1 2; do echo -n "$T: "; UB_LIB=$LIBF timeout 60 python scripts/probe_time.py; done
done
