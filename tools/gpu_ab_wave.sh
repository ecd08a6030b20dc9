# A/B: wave-engine geometry (register model) variants built under abtmp*/
S=8,16,24,32,40,48,56,64,72,80,88,96,104,112,120,128
for root in ${ROOTS:-.}; do
  for eq in sylvester:13 lyapunov:5; do
    LAGEN_PKG_ROOT=$root timeout 300 python tools/engine_compare.py --eq ${eq%%:*} --sizes $S --runs ${eq##*:}:8:wave --reps 3 | sed "s/^/$root /"
  done
done > gpurun_out/ab_wave.txt 2>&1
