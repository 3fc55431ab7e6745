#!/bin/bash
# fit_modes.py for each given libgi variant
cp paper_2403_08551_b200/libgi.so /tmp/libgi_orig.so
for V in "$@"; do cp $V paper_2403_08551_b200/libgi.so; echo "== $V"; python tools/fit_modes.py 2>&1 | grep chained; done
cp /tmp/libgi_orig.so paper_2403_08551_b200/libgi.so
