#!/bin/bash
# Build libhermb200.so with extra compile-time knobs into build_var/<name>/, for
# A/B timing against the default build:
#   tools/build_variant.sh nowres -DHW_CM_WRES=0
#   HERMB200_LIB=build_var/nowres/libhermb200.so python tools/prof_step.py ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build_var/$name
mkdir -p $out
make -s -j12 BUILD=$out LIB=$out/libhermb200.so EXTRA="$*" $out/libhermb200.so
