for a in "sylvester 68 13" "sylvester 128 13" "lyapunov 92 5" "lyapunov 64 5"; do set -- $a
  python tools/run_one.py --eq $1 --n $2 --variant $3 --b 4 --engine wave --reps 3 2>&1 | tail -1
done
CMD="python tools/run_one.py --eq sylvester --n 68 --variant 13 --b 4 --engine wave --reps 1"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:wave --csv $CMD 2>/dev/null | grep -E "dram|duration" | tail -3
