o=gpurun_out/r02x; mkdir -p $o
# r02x (historical): ncu of the per-line L2 prefetch variants 2/4 of the cells kernel
# (applied from a working copy, then removed) -> profiles/r02/r02x_ncu_cells_prefetch_negative.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:mttkrp_cells -c 3 --csv --log-file $o/ncu.csv python tools/sweep_cells.py --config cfg2 --modes 0 --reps 0 --specs '[{"variant":1},{"variant":2},{"variant":4}]' > $o/ncu.log 2>&1
