#!/bin/bash
# Static SASS statistics of one kernel: FP64 / local-memory / global-load instruction counts.
# usage: tools/sass_stats.sh <source.cu> <mangled-kernel-name> [extra nvcc flags]
SRC=$1; FN=$2; shift 2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include "$@" -cubin -o /tmp/_stats.cubin "$SRC" || exit 1
cuobjdump -sass -fun "$FN" /tmp/_stats.cubin > /tmp/_stats.sass
printf "instr %s  DFMA %s  DMUL/DADD %s  MUFU %s  STL %s  LDL %s  LDG %s\n" \
  "$(grep -cE '^\s+/\*[0-9a-f]{4,5}\*/' /tmp/_stats.sass)" "$(grep -c DFMA /tmp/_stats.sass)" \
  "$(grep -cE 'DMUL|DADD' /tmp/_stats.sass)" "$(grep -c MUFU /tmp/_stats.sass)" "$(grep -c STL /tmp/_stats.sass)" \
  "$(grep -c LDL /tmp/_stats.sass)" "$(grep -c LDG /tmp/_stats.sass)"
