#!/bin/bash
# c3_probe.py (CFG=C2 and C3) for each given libgi variant
cp paper_2403_08551_b200/libgi.so /tmp/libgi_orig.so
for V in "$@"; do cp $V paper_2403_08551_b200/libgi.so; for C in C2 C3; do echo "== $V $C"; CFG=$C python tools/c3_probe.py 2>&1 | grep config; done; done
cp /tmp/libgi_orig.so paper_2403_08551_b200/libgi.so
