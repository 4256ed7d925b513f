#!/bin/bash
# Counter matrix for tools/randbw_matrix.cu (run under gpurun; writes gpurun_out/).
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__sectors_read.sum,dram__bytes_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
tools/randbw_matrix 32 > gpurun_out/randbw_matrix.log 2>&1
ncu --clock-control none --metrics $M --csv --log-file gpurun_out/randbw_matrix_ncu.csv tools/randbw_matrix 32 1 > gpurun_out/randbw_matrix_ncu.log 2>&1
