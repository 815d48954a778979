#!/bin/bash
# The put over NVLink from one process (scripts/put_nvlink.py), then ncu --set
# full of rank 0's put kernel and of the p2pbench TMA push kernel (single
# process: no rank waits on a profiled peer).
o=gpurun_out/nvl; mkdir -p $o
timeout 300 python scripts/put_nvlink.py 2 > $o/put_nvlink_2.log 2>&1; echo "put 2 rc=$? $(tail -2 $o/put_nvlink_2.log | tr '\n' ' ')"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_move_tma -c 1 -o $o/put_full \
  python scripts/put_nvlink.py 2 --no-barrier > $o/put_ncu.log 2>&1; echo "ncu put rc=$?"
timeout 300 ncu --set full --clock-control none -k regex:k_tma -s 2 -c 1 -o $o/p2p_tma_full \
  paper_2503_23830_b200/lib/p2pbench 256 tma uni > $o/p2p_ncu.log 2>&1; echo "ncu p2p rc=$?"
