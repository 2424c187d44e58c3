#!/bin/bash
# Round-end measurement set (run under gpurun): bench.py on every BASELINE config, the reference arm,
# the launch list of the default run, and one ncu --set full capture of the dominant kernel.
O=gpurun_out/final_r02
mkdir -p $O
python bench.py > $O/cfg2.json 2> $O/cfg2.err
for c in 1 3 4; do python bench.py --config $c --steps 200 > $O/cfg$c.json 2> $O/cfg$c.err; done
python bench.py --config 5 --steps 20 --warmup 3 > $O/cfg5.json 2> $O/cfg5.err
python bench.py --impl reference --steps 20 --warmup 3 > $O/ref_cfg2.json 2> $O/ref_cfg2.err
python bench.py --steps 20 --warmup 3 --no-formats --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --steps 20 --warmup 3 --no-formats --no-cpu > $O/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:merge_hot --launch-skip 5 -c 1 -o $O/merge_hot -f \
  python bench.py --steps 20 --warmup 3 --no-formats --no-cpu > $O/ncu_full.log 2>&1
tail -n 2 $O/*.err
