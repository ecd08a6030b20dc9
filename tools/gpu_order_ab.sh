# A/B of the rows-engine problem order at BASELINE config 5 (n = 64, 2^20 problems):
# abtmp/ = CTA-major (-DLAGEN_ROWS_SPREAD=0), . = slot-major; time + DRAM bytes per launch
for root in abtmp .; do
  LAGEN_PKG_ROOT=$root timeout 300 python tools/engine_compare.py --eq cholesky --sizes 64 --runs 1:8:rows --bytes 34359738368 --reps 3 | sed "s|^|$root |"
  LAGEN_PKG_ROOT=$root timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:chol_rows_kernel -c 1 --csv \
     python tools/engine_compare.py --eq cholesky --sizes 64 --runs 1:8:rows --bytes 34359738368 --reps 1 2>&1 | grep -E '"(gpu__time|dram__|lts__)' | sed "s|^|$root |"
done > gpurun_out/order_ab.txt 2>&1
