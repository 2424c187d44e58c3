# dev: one ncu --set full capture of the merge kernel (hot plan) on cfg2
ncu --set full --import-source on --clock-control none -k regex:merge_hot --launch-skip 3 -c 1 -o gpurun_out/hot_merge -f python tools/hot_merge_probe.py 2 "${1:-}" > gpurun_out/ncu2.log 2>&1
tail -n 3 gpurun_out/ncu2.log
