#!/bin/bash
# knock-out sweep: step time with each kernel family skipped (results wrong; timing only)
TAG=${1:-r3f}
O=gpurun_out
timeout 300 python tools/graph_kernel_times.py > $O/${TAG}_graph_kernel_times.txt 2>&1
for k in "" k_aggregate k_aggregate_combine k_csc_backward k_csc_dots k_csc_combine k_umma_gemm_nn k_umma_gemm_tn \
         k_umma_pack k_score k_sub_partials k_group_finish k_dz k_dense_step k_sparse_step k_pack_weights \
         k_copy_segments k_csc_positions k_dcoeff_reduce,k_dcoeff_final; do
  echo "$k $(KG_KNOCKOUT=$k timeout 120 python tools/knockout.py 2>/dev/null | tail -1)" >> $O/${TAG}_knockout.txt
done
