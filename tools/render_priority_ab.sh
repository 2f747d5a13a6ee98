for r in 1 2; do for c in c2 c3 c1; do for k in 0 1; do NGS_RENDER_PRIORITY=$k python tools/step_profile.py $c 5 2>&1 | grep -E "concurrent steps" | sed "s/^/rp$k: /"; done; done; done
