#!/bin/bash
# round-2 final evidence, part B: bench lines for every config and path on the final kernels (clocks included)
mkdir -p gpurun_out/r02
O=gpurun_out/r02
B="timeout 400 python bench.py"
Q="--no-e2e --no-cpu-baseline"
$B --steps 20 --warmup 5 > $O/bench_default.jsonl 2> $O/bench_default.err
for c in C1 C2; do $B --config $c --graph 100 --steps 20 --warmup 5 $Q > $O/bench_$c.jsonl 2> $O/bench_$c.err; done
$B --config C3 --steps 10 --warmup 3 $Q > $O/bench_C3.jsonl 2> $O/bench_C3.err
$B --config C5 --steps 3 --warmup 1 $Q > $O/bench_C5_whole.jsonl 2> $O/bench_C5_whole.err
$B --config C5 --slab 0/8 --steps 5 --warmup 3 $Q > $O/bench_C5_slab0of8.jsonl 2> $O/bench_C5_slab0of8.err
for c in C3 C4; do $B --config $c --path adjoint --steps 10 --warmup 3 $Q > $O/bench_adjoint_$c.jsonl 2> $O/bench_adjoint_$c.err; done
$B --config C4 --degree 4 --steps 5 --warmup 3 $Q > $O/bench_C4_p4.jsonl 2> $O/bench_C4_p4.err
$B --config C4 --degree 4 --path adjoint --steps 10 --warmup 3 $Q > $O/bench_adjoint_C4_p4.jsonl 2> $O/bench_adjoint_C4_p4.err
for c in C2 C3 C4; do $B --config $c --path saved --steps 10 --warmup 3 $Q > $O/bench_saved_$c.jsonl 2> $O/bench_saved_$c.err; done
for c in C2 C4; do
  $B --config $c --path fused --steps 10 --warmup 3 $Q > $O/bench_${c}_fused.jsonl 2> $O/bench_${c}_fused.err
  $B --config $c --steps 10 --warmup 3 $Q > $O/bench_${c}_primal.jsonl 2> $O/bench_${c}_primal.err
done
for c in C2 C3 C4; do $B --config $c --path solve --steps 2 --warmup 1 $Q > $O/bench_solve_$c.jsonl 2> $O/bench_solve_$c.err; done
HDG_CONDENSE_KERNEL=rows $B --config C3 --steps 5 --warmup 3 $Q > $O/bench_rows_C3.jsonl 2> $O/bench_rows_C3.err
HDG_CONDENSE_KERNEL=rows $B --config C4 --steps 5 --warmup 3 $Q > $O/bench_rows_C4.jsonl 2> $O/bench_rows_C4.err
