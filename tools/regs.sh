#!/bin/bash
# Register / spill report of one instantiation unit: tools/regs.sh K PART [extra nvcc flags]
K=$1; PART=$2; shift 2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false --expt-relaxed-constexpr \
  -I include -I paper_2510_16172_b200/csrc -Xptxas -v "$@" -c paper_2510_16172_b200/csrc/fp_inst.cu \
  -DFP_INST_K=$K -DFP_INST_PART=$PART -o /tmp/regs_$$.o 2>&1 \
  | grep -E "Compiling entry|Used|spill" | paste - - - \
  | sed -E 's/.*path_kernelI([fd])Li([0-9]+)ELj([0-9]+)ELi([0-9])E.*bytes stack frame, ([0-9]+) bytes spill stores, ([0-9]+) bytes spill loads.*Used ([0-9]+) registers.*/\1 K=\2 mask=\3 op=\4 regs=\7 spill_st=\5 spill_ld=\6/'
rm -f /tmp/regs_$$.o
