#!/bin/bash
# Compile only the production fused SMPC kernel (smpc_kernel<float, float, 8, TopoRobot7>)
# for register / spill / SASS inspection: tools/quick_sass.sh [extra nvcc flags]
# -> /tmp/vpb_quick.o, /tmp/vpb_quick.sass, ptxas summary on stdout.
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Iinclude \
  -DVPB_QUICK -Xptxas -v "$@" -c paper_2512_22575_b200/csrc/rollout.cu -o /tmp/vpb_quick.o 2>&1 \
  | grep -A2 "Compiling entry function '_ZN3vpb11smpc_kernelIffLi8ENS_10TopoRobot7ELb0" | tail -2
cuobjdump -sass -fun '_ZN3vpb11smpc_kernelIffLi8ENS_10TopoRobot7ELb0EEEvNS_4ProbIT_EENS_6SmpcIOENS_9NomInlineIXT3_EEE' /tmp/vpb_quick.o > /tmp/vpb_quick.sass
echo "sass lines: $(grep -c '^        /\*[0-9a-f]*\*/' /tmp/vpb_quick.sass)  LDL: $(grep -c LDL /tmp/vpb_quick.sass)  STL: $(grep -c STL /tmp/vpb_quick.sass)"
