# attn_one.cu ablations: K1 at ADASPA_ONE=1 (full), 2 (no softmax), 3 (no exponentials), and the
# default kernel.  Timing only (ablations are not correct).
cd "$GRAFT_REPO_ROOT" || exit 1
for m in 2 3 4; do echo "ADASPA_ONE=$m"; ADASPA_ONE=$m timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep "K1"; done
timeout 120 python tools/quick_timing.py hyv110k 2>&1 | grep "K1"
