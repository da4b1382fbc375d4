# usage (GPU box): bash scripts/gpu_ncu_gather.sh TAG — key memory metrics of one warm contraction + gather (C4)
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-g}
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_write.sum,launch__shared_mem_config_size,sm__warps_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 2 -c 2 \
  python bench.py --profile-only --steps 1 --warmup 0 2>&1 | grep -E "__|gather_fast|partial_contract" | grep -v "==PROF" > gpurun_out/ncu_mem_$TAG.txt
cat gpurun_out/ncu_mem_$TAG.txt
