#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02ak; mkdir -p $O
FMMGPU_AUX=0 timeout 600 python tools/scratch/rank_probe.py 8 > $O/rank8_aux0.txt 2>&1
FMMGPU_AUX=1 timeout 600 python tools/scratch/rank_probe.py 8 > $O/rank8_aux1.txt 2>&1
head -1 $O/rank8_aux0.txt $O/rank8_aux1.txt; cat $O/rank8_aux0.txt | tail -30
