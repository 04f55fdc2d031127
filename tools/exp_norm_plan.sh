#!/bin/bash
# 8K detect (pad) normalize / clamp_abs over kernel U's plan knobs (pairs per
# lane, warps per CTA, band rows): does the S mode (normalize pass 1) want a
# different plan from clamp_abs?  tools/detect_time.py, CUDA events.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for np in 4 2; do for w in 2 4 1; do for b in 16 24 32 8; do
  echo "np $np warps $w band $b: $(SOBEL5_U8_NP=$np SOBEL5_U8_WARPS=$w SOBEL5_U8_BAND=$b python tools/detect_time.py | tr '\n' ' ')"
done; done; done
