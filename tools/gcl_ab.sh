# gcl Jacobi phase timing: default plan and forced cluster sizes, full vs cross-pair block rounds
for x in 0 1; do for C in "" 4 8 16; do echo "CROSS=$x C=$C"; RSVD_GCL_CROSS=$x ${C:+RSVD_GCL_C=$C} ./tools/gcl_probe 70 140 250 500 2>&1 | grep "J=0"; done; done
