#!/bin/bash
# dev: ncu --set full of the other hot kernels at cfg2 (one launch each): one onesweep pass of the
# CRS conversion, the blocked (MergeB) and window (CSB) multiplies
O=gpurun_out/r02x
mkdir -p $O
ncu --set full --clock-control none -k regex:rs_onesweep -s 6 -c 1 -o $O/onesweep -f python tools/quick_spmv.py 22 2 > $O/onesweep.log 2>&1
ncu --set full --clock-control none -k regex:"blocked_spmv|window_spmv" -c 2 -o $O/blocked -f python tools/probe_blocked.py 22 9,3 > $O/blocked.log 2>&1
tail -n 2 $O/*.log
