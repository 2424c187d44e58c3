#!/bin/bash
# The CPU reference baseline at cfg2 on the GPU box's host cores (run under gpurun; ~1 h).
set -x
O=gpurun_out/cpu_ref
mkdir -p $O
free -g > $O/free.txt; nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
python tools/cpu_reference_bench.py 2 spmv --algs 1,2 --threads 1,2,4,8,16 --spmv-reps 100 --out $O/cfg2_spmv_psweep.json
python tools/cpu_reference_bench.py 2 spmv --spmv-reps 550 --out $O/cfg2_spmv_all.json
python tools/cpu_reference_bench.py 2 convert --convert-reps 1 --spmv-reps 100 --out $O/cfg2_convert_all.json
