#!/bin/bash
# dev: full GPU tests, the default bench line, and one ncu --set full capture of the merge kernel
O=gpurun_out/r03
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/gputests.log 2>&1; echo "pytest rc=$?" >> $O/gputests.log
timeout 600 python bench.py --no-cpu > $O/cfg2.json 2> $O/cfg2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_hot --launch-skip 5 -c 1 -o $O/merge_hot -f \
  python bench.py --steps 20 --warmup 3 --no-formats --no-cpu > $O/ncu.log 2>&1
tail -n 3 $O/gputests.log; tail -c 600 $O/cfg2.json
