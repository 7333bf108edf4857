# ncu metrics of the merge gathers of one L=8 build (developer tool): bash tools/gather_prof.sh [LIB] [TAG]
cd ${GRAFT_REPO_ROOT:-.}
LIB=${1:-paper_2503_17535_b200/libhps_b200.so}; TAG=${2:-cur}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum -k regex:gather_kernel -c 22 --csv --log-file gpurun_out/gather_metrics_$TAG.csv python tools/solve_ab.py $LIB /tmp/u.npy > gpurun_out/gp_$TAG.log 2>&1
echo done $?
