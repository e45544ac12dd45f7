#!/usr/bin/env bash
#   gpurun --timeout 3600 -- 'bash tools/gpu_evidence.sh <tag>'
# Evidence on the current build: steady-state per-launch DRAM traffic (no
# cache flush: the previous launch's write-backs land in this one), graph-level
# per-iteration traffic, ncu full of the step kernels (transport, PageRank-10M
# dual with the gather sweep) summarised on the box, the bench launch list,
# the bench line and the reference arm.
O=gpurun_out/${1:-evidence}; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --cache-control none --clock-control none -k regex:"OpPrimal|OpDual" -c 120 --csv --log-file $O/steady_transport.csv python tools/profile_step.py transport - 64 > $O/steady_transport.log 2>&1
timeout 600 ncu --graph-profiling graph --metrics $M --cache-control none --clock-control none --csv --log-file $O/graph_transport.csv python tools/profile_step.py transport - 64 > $O/graph_transport.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"OpDual|OpPrimal" -c 4 -o /tmp/ncu_transport python tools/profile_step.py transport > $O/ncu_transport.log 2>&1
python tools/ncu_summary.py full /tmp/ncu_transport.ncu-rep --json $O/ncu_full_transport.json > $O/ncu_full_transport.md 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"OpDual" -c 5 -o /tmp/ncu_pr10m python tools/profile_step.py pagerank 10000000 2 > $O/ncu_pr10m.log 2>&1
python tools/ncu_summary.py full /tmp/ncu_pr10m.ncu-rep --json $O/ncu_full_pr10m_dual.json > $O/ncu_full_pr10m_dual.md 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 1 --kernel-iters 8 --extra "" > $O/launches_bench.log 2>&1
python tools/ncu_summary.py launches /tmp/launches.csv --json $O/launches.json > $O/launches.md 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
du -sh $O
echo done
