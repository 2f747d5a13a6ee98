L=paper_2501_13975_b200/lib
for v in cf3 cf4 cf5; do python tools/solve_mb.py $L/$v.so; done
NGS_COLOR_FUSED=0 python tools/solve_mb.py $L/cf4.so
