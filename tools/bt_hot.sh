python tools/build_timing.py 22 2
SPMVLAB_MERGE_HOT=0 python tools/build_timing.py 22 2
SPMVLAB_MERGE_HOT_SLOTS=1 python tools/build_timing.py 22 2
