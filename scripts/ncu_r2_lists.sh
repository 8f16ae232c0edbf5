#!/bin/bash
# full ncu capture of the list kernels (c4 @ 2^26), one steady-state launch each; only text summaries are kept
mkdir -p gpurun_out
TAG=${TAG:-r2n}
KERNELS=${KERNELS:-"k_list_build k_list_scan k_list_forces"}
CMD="python bench.py --steps 14 --warmup 3 --no-cpu --no-e2e"
for k in $KERNELS; do
  skip=8; [ $k = k_list_build ] && skip=2; [ $k = k_force ] && skip=2
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^$k -s $skip -c 1 -o /tmp/${TAG}_$k -f $CMD > gpurun_out/${TAG}_ncu_$k.log 2>&1
  ncu -i /tmp/${TAG}_$k.ncu-rep --page details > gpurun_out/${TAG}_${k}_details.txt 2>/dev/null
  ncu -i /tmp/${TAG}_$k.ncu-rep --page raw --csv > /tmp/${TAG}_${k}_raw.csv 2>/dev/null
  python - <<PY > gpurun_out/${TAG}_${k}_raw_sel.txt
import csv
rows=list(csv.reader(open("/tmp/${TAG}_${k}_raw.csv")))
h,u,v=rows[0],rows[1],rows[2]
keys=["gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","smsp__inst_executed.sum","smsp__thread_inst_executed.sum","sm__warps_active.avg.pct_of_peak_sustained_active","smsp__issue_active.avg.pct","l1tex__t_sector_hit_rate.pct","lts__t_sector_hit_rate.pct","launch__registers_per_thread","launch__grid_size","launch__block_size","l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum","l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum","lts__t_sectors_srcunit_tex_op_read.sum","smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio","smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio","smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_wait_per_issue_active.ratio","smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio","smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio","smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio","smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio","smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio","smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio","smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio","smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio","sm__inst_executed_pipe_fp64.sum","sm__inst_executed_pipe_lsu.sum","sm__inst_executed_pipe_fma.sum","sm__inst_executed_pipe_alu.sum","smsp__thread_inst_executed_per_inst_executed.ratio","lts__t_bytes.sum","l1tex__t_bytes.sum","l1tex__data_pipe_lsu_wavefronts.sum","sm__throughput.avg.pct_of_peak_sustained_elapsed","l1tex__throughput.avg.pct_of_peak_sustained_elapsed","lts__throughput.avg.pct_of_peak_sustained_elapsed","dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for i,n in enumerate(h):
    if n in keys or n in ("Kernel Name",): print(n, u[i], v[i])
PY
  ncu -i /tmp/${TAG}_$k.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${TAG}_${k}_source.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/${TAG}_${k}_source.csv 45 > gpurun_out/${TAG}_${k}_lines.txt 2>&1
  echo "== $k"; grep -E "Duration|Registers Per|Achieved Occupancy|Executed Ipc Active|Issue Slots Busy|L1/TEX Hit|L2 Hit|DRAM Throughput" gpurun_out/${TAG}_${k}_details.txt | head -9
  rm -f /tmp/${TAG}_$k.ncu-rep /tmp/${TAG}_${k}_raw.csv /tmp/${TAG}_${k}_source.csv
done
