#!/bin/bash
# run phase_timing.py against the FKS_TIMING build (tools/libfks_timing.so)
cp paper_1608_08009_b200/libfks.so /tmp/libfks_keep.so
cp tools/libfks_timing.so paper_1608_08009_b200/libfks.so
python tools/phase_timing.py
cp /tmp/libfks_keep.so paper_1608_08009_b200/libfks.so
