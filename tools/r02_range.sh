#!/bin/bash
# GPU-wide counters of the pipelined render (tools/range_prof.py) at C3 and C4
mkdir -p gpurun_out/r02range
python -m paper_2503_16422_b200.build > gpurun_out/r02range/build.log 2>&1
M=sm__cycles_active.avg,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,smsp__warps_issue_stalled_long_scoreboard.avg,smsp__warps_issue_stalled_barrier.avg,smsp__warps_issue_stalled_wait.avg,smsp__warps_issue_stalled_membar.avg,smsp__warps_issue_stalled_lg_throttle.avg,smsp__warps_issue_stalled_short_scoreboard.avg,smsp__warps_issue_stalled_math_pipe_throttle.avg,smsp__warps_issue_stalled_no_instruction.avg,smsp__warps_issue_stalled_sleeping.avg,smsp__warps_issue_stalled_drain.avg,smsp__warps_issue_stalled_mio_throttle.avg,smsp__warps_issue_stalled_branch_resolving.avg,smsp__warps_issue_stalled_not_selected.avg,smsp__warps_issue_stalled_selected.avg,smsp__warps_issue_stalled_dispatch_stall.avg,sm__ctas_launched.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum
for c in c3 c4; do
  python tools/range_prof.py --config $c > gpurun_out/r02range/plain_$c.log 2>&1 && \
  ncu --replay-mode app-range --clock-control none --metrics $M --csv --log-file gpurun_out/r02range/range_$c.csv python tools/range_prof.py --config $c > gpurun_out/r02range/ncu_$c.log 2>&1
  echo "$c rc=$?"
done
