#!/bin/bash
# stage times of variant libraries: exp/ab_stages.sh lib1 lib2 ...  (B from env, default 128)
for L in "$@"; do
  for rep in 1 2; do SGL_B200_LIB=$PWD/$L timeout 100 python exp/stage_time.py; done
done
