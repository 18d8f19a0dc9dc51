python tools/time_calls.py 4 100000000 3 16 2>&1 | tail -2
timeout 1500 python tools/full_size.py 5 > gpurun_out/r2_full_c5.jsonl 2> gpurun_out/r2_full_c5.err; tail -3 gpurun_out/r2_full_c5.err; cat gpurun_out/r2_full_c5.jsonl
