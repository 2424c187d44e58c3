# dev: ncu of blocked_spmv_kernel (MergeB) at cfg3 with the L2 breakdown by operation
ncu --section MemoryWorkloadAnalysis_Tables --section MemoryWorkloadAnalysis --section SpeedOfLight \
    --metrics lts__t_sectors_op_read.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,lts__t_sector_op_write_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:blocked_spmv -c 1 -o gpurun_out/blk_c3 -f python tools/engine_time.py 3 9 > gpurun_out/blk_c3.log 2>&1
tail -n 3 gpurun_out/blk_c3.log
