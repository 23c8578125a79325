#!/bin/bash
# compile csrc/batched_pipe.cu alone: registers / spills and the code size of each warp role
cd /root/repo/paper_1002_4057_b200/csrc || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -c batched_pipe.cu -o /tmp/bp.o -Xptxas -v 2>&1 | grep -E "error|spill|Used" | tail -2
cuobjdump -sass /tmp/bp.o | awk '/Function : _ZN4tinv3bpl7k_bpipeILb0/{f=1} f' | grep -E "USETMAXREG|EXIT ;" | awk '{print $1, $2, $3}'
