cd "${GRAFT_REPO_ROOT:-/root/repo}"
for b in 4 8 16 32; do echo "band $b"; W=1920 H=1080 CONTRACT=u8 BANDS=$b python tools/sweep.py | tail -1; W=3840 H=2160 CONTRACT=u8 BANDS=$b python tools/sweep.py | tail -1; W=1920 H=1080 CONTRACT=sr BANDS=$b python tools/sweep.py | tail -1; W=3840 H=2160 CONTRACT=sr BANDS=$b python tools/sweep.py | tail -1; done
