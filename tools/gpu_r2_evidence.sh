#!/bin/bash
# round-2 evidence: bench lines for every config and path (clocks included), default line with e2e/cpu_baseline
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi -L > $O/smi.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.jsonl 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.jsonl 2> $O/bench_reference.err
for c in C1 C2; do timeout 600 python bench.py --config $c --graph 100 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_$c.jsonl 2> $O/bench_$c.err; done
for c in C3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.jsonl 2> $O/bench_$c.err; done
timeout 900 python bench.py --config C5 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_C5_whole.jsonl 2> $O/bench_C5_whole.err
timeout 600 python bench.py --config C5 --slab 0/8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5_slab0of8.jsonl 2> $O/bench_C5_slab0of8.err
for c in C3 C4; do timeout 600 python bench.py --config $c --path adjoint --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_adjoint_$c.jsonl 2> $O/bench_adjoint_$c.err; done
timeout 600 python bench.py --config C4 --path saved --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_saved_C4.jsonl 2> $O/bench_saved_C4.err
HDG_CONDENSE_KERNEL=rows timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_rows_C3.jsonl 2> $O/bench_rows_C3.err
HDG_CONDENSE_KERNEL=rows timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_rows_C4.jsonl 2> $O/bench_rows_C4.err
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/r02/bench_*.jsonl")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "ERR", open(f.replace('.jsonl', '.err')).read()[-300:]); continue
    keys = ("value", "ms_per_step", "condense_ms", "assemble_ms", "backsub_ms", "save_solutions_ms", "exchange_ms",
            "adjoint_rhs_ms", "backsub_adjoint_ms")
    print(os.path.basename(f), {k: round(d[k], 4) for k in keys if isinstance(d.get(k), (int, float))},
          "frac", round(d.get("roofline", {}).get("frac", 0) or 0, 3), "graph", (d.get("cuda_graph") or {}).get("ms_per_step"),
          "clk", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
PY
