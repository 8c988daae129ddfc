#!/bin/bash
# L2-residency experiment for G: default build vs L2 eviction hints, unsliced vs shell slices.
cd $GRAFT_REPO_ROOT
H=$PWD/exp/lib_hints.so
bash exp/sweep.sh l2 "SGL_G_CHUNK_MB=0" "SGL_G_CHUNK_MB=32" "SGL_G_CHUNK_MB=16" "SGL_B200_LIB=$H SGL_G_CHUNK_MB=0" "SGL_B200_LIB=$H SGL_G_CHUNK_MB=32" "SGL_B200_LIB=$H SGL_G_CHUNK_MB=16" "SGL_B200_LIB=$H SGL_G_CHUNK_MB=64"
