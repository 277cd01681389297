for l in phase p1a p1b p1c; do cp tools/diag/sweep/lib_$l.so tools/diag/libhdg_b200_phase.so; echo "== $l"; timeout 200 python tools/diag/phase_timing.py C2 3 2>&1 | head -3; done
