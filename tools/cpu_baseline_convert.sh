#!/bin/bash
# The CPU reference conversions at cfg2 (bench_convert, one repetition per engine) and sampled
# cfg3 / cfg4 multiplies, on the GPU box's host cores (run under gpurun).
set -x
O=gpurun_out/cpu_ref
mkdir -p $O
python tools/cpu_reference_bench.py 2 convert --convert-reps 1 --spmv-reps 20 --out $O/cfg2_convert_all.json
python tools/cpu_reference_bench.py 3 spmv --algs 1,2,6,9 --spmv-reps 20 --out $O/cfg3_spmv_sample.json
python tools/cpu_reference_bench.py 4 spmv --algs 1,2,6,9 --spmv-reps 20 --out $O/cfg4_spmv_sample.json
