for i in 1 2; do for v in 0 1; do echo "UPD_CP16=$v"; RQB_UPD_CP16=$v timeout 300 python tools/dag_prof.py cfg2_riga cfg4_riga cfg4_iga | grep "factor"; done; done
