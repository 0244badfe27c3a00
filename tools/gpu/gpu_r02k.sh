#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02k; mkdir -p $O
timeout 300 python tools/scratch/twin_probe.py > $O/twin.txt 2>&1
FMMGPU_P2P_ONESIDED=1 timeout 300 python tools/scratch/twin_probe.py > $O/twin_onesided.txt 2>&1
cat $O/*.txt
