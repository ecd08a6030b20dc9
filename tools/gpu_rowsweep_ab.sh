for eq in lyapunov sylvester; do v=5; [ $eq = sylvester ] && v=13
timeout 300 python tools/engine_compare.py --eq $eq --sizes 4,8,12,16,20,24,28,32 --runs $v:4:generic,$v:0:rowsweep --reps 5
done
