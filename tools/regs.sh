#!/bin/bash
# registers / spills of the hot kernels from build_ptxas.log
grep -A3 "Compiling entry function" build_ptxas.log | grep -E "entry|Used|spill" | paste - - - | \
  sed -E "s/.*entry function '([^']*)'.*([0-9]+ bytes spill stores, [0-9]+ bytes spill loads).*Used ([0-9]+) registers.*/\3 regs  \2  \1/" | \
  grep -E "bjac_tile|spmv|update|k_resid" | c++filt | sort -u
