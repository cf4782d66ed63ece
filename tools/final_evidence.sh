#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
# GPU suite, smoke, bench line, C1..C5 configs, ncu launch list of one bench
# step, a full ncu capture and bench-size counters of the dominant kernel,
# full-size parity runs and the device-assert build's suite.
# Everything lands in gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
python bench.py > $O/bench.jsonl 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.jsonl 2> $O/bench_reference.err
timeout 900 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mc_stats_mma -s 1 -c 1 \
    -o $O/k_mc_stats_mma python tools/profile_mc.py 2097152 > $O/ncu_full.log 2>&1
M="dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum"
timeout 900 ncu --metrics $M --clock-control none -k regex:k_mc_stats_mma -s 1 -c 1 --csv --log-file $O/bench_kernel.csv \
    python tools/profile_mc.py 100000000 > $O/bench_kernel.log 2>&1
for c in c2 c3 c4 c5; do timeout 900 python tests/parity/full_parity.py $c > $O/full_parity_$c.json 2> $O/full_parity_$c.err; done
FRR_LIBRARY=tools/variants/libfrr_checks.so timeout 1500 python -m pytest tests -m gpu -q > $O/checks_gpu_tests.txt 2>&1
FRR_LIBRARY=tools/variants/libfrr_checks.so timeout 900 python tests/parity/sanitize.py > $O/checks_sanitize.txt 2>&1
for f in gpu_tests.txt checks_gpu_tests.txt smoke.txt; do tail -n 1 $O/$f; done
