# rows / padded-rows timing + sampled oracle check at full batches (no pytest)
timeout 300 python tools/rows_check.py --sizes ${S:-36,40,44,48,52,56,60,64,68,72,76,80,84,88,92,96,100,104,108,112,116,120,124,128} > gpurun_out/rows_check.jsonl 2>&1
