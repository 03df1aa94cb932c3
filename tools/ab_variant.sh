#!/bin/bash
# Developer A/B builds: a complete, consistent libsbg in ablibs/ with extra nvcc flags (objects in
# their own build directory), e.g. one k-step count of K6 so the build takes seconds.
#   tools/ab_variant.sh <name> "<nvcc flags>"      e.g.  tools/ab_variant.sh x16 "-DSBG_KS_ONLY=16"
#   SBG_LIB_PATH=ablibs/libsbg_<name>.so python tools/sigma_modes.py c4
set -e
cd "$(dirname "$0")/.."
mkdir -p ablibs
SBG_NVCC_FLAGS="$2" SBG_LIB_OUT=$PWD/ablibs/libsbg_$1.so python -m paper_2603_06101_b200.build --force
