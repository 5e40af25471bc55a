mkdir -p gpurun_out
timeout 900 python tools/bench_rows.py > gpurun_out/r2_rows.jsonl 2> gpurun_out/r2_rows.err; echo rows=$?
cat gpurun_out/r2_rows.jsonl | cut -c1-400
tail -3 gpurun_out/r2_rows.err
