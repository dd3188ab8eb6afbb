# A/B of the 3xTF32 A split: truncation (default, A_hi implicit) vs rounded (RSVD_TF32_RNA=1)
for r in 1 0; do echo "RSVD_TF32_RNA=$r"; RSVD_TF32_RNA=$r python tools/tf32_bias_probe.py 2>&1 | grep -v Warn | tail -6; done
