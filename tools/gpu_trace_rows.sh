#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/trace_rows.py --config C4 --nr 32 --nt 64 --show 90 > gpurun_out/trace_rows_C4.txt 2>&1
timeout 300 python tools/trace_rows.py --config C3 --nr 64 --nt 64 --show 60 > gpurun_out/trace_rows_C3.txt 2>&1
head -5 gpurun_out/trace_rows_C4.txt; tail -4 gpurun_out/trace_rows_C4.txt; tail -3 gpurun_out/trace_rows_C3.txt
