P=paper_2112_14064_b200
for i in 1 2; do for v in old new; do cp $P/librq_$v.so $P/librq_b200.so; echo $v; for c in cfg4_riga cfg4_iga; do timeout 100 python tools/solve_prof.py $c | tail -1; done; done; done
