echo "== d=71 fused"; timeout 300 python tools/quick_time.py 71 71 4 2>&1 | grep -v phases | tail -3
echo "== d=71 unfused"; SK_FUSE_COLS=0 timeout 300 python tools/quick_time.py 71 71 4 2>&1 | grep -v phases | tail -3
