for w in 128 64 32 16 8 4; do echo "WHOLE_MIN=$w"; RQB_WHOLE_MIN=$w timeout 120 python tools/solve_prof.py cfg2_riga 2>&1 | tail -1; done
for w in 256 128 64; do echo "WHOLE_MIN=$w"; RQB_WHOLE_MIN=$w timeout 200 python tools/solve_prof.py cfg4_riga 2>&1 | tail -1; RQB_WHOLE_MIN=$w timeout 200 python tools/solve_prof.py cfg3_riga 2>&1 | tail -1; done
