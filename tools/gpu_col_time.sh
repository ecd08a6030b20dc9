# column-engine timing at full batches (variants 1 and 2, b = 4)
timeout 300 python tools/engine_compare.py --eq cholesky --sizes ${S:-20,24,28,32} --runs 1:4:column,2:4:column --reps 5 > gpurun_out/col_time.jsonl 2>&1
