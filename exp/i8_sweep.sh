#!/bin/bash
# stage times, DMMA vs INT8 Legendre inverse, tiles-per-CTA sweep
for B in 128 256 64; do
  echo "== B=$B"
  B=$B SGL_I8=0 timeout 120 python exp/stage_time.py
  for tpc in 1 2 4 8; do echo "tpc=$tpc"; B=$B SGL_I8=leginv SGL_I8_TPC=$tpc timeout 120 python exp/stage_time.py; done
done
