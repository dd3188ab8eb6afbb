# core SVD time by forced cluster size (RSVD_GCL_C) for the gcl widths
for C in 4 8 16; do echo "C=$C"; RSVD_GCL_C=$C python tools/core_probe.py 70 140 250 2>&1 | grep "noJ"; done
