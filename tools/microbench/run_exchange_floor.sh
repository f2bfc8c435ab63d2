#!/bin/bash
# Exchange / barrier floors behind the LUPP pivot-step latency (run on the GPU box):
# DSMEM all-to-all rounds in a 16-CTA cluster, cluster.sync / grid.sync / __syncthreads, and
# grid.sync plus a per-step candidate exchange through global memory at the panel-LUPP shapes.
set -e
cd "$(dirname "$0")"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17"
mkdir -p /tmp/mb
for b in dsmem_bench sync_bench gridsync; do $NV $b.cu -o /tmp/mb/$b; done
for b in dsmem_bench sync_bench gridsync; do echo "== $b"; /tmp/mb/$b; done
