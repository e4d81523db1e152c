# block Krylov-Schur sweep (development aid): time to nev per block size on cfg4_riga / cfg3_riga
for ms in ${MINSTEPS:-1}; do
  echo "== minsteps $ms"
  RQB_BLOCK_MINSTEPS=$ms timeout 300 python tools/block_trace.py cfg4_riga 100 ${BLOCKS:-2,4,8} 100 2>/dev/null | grep "run 1"
  RQB_BLOCK_MINSTEPS=$ms timeout 300 python tools/block_trace.py cfg3_riga 50 ${BLOCKS:-2,4,8} 100 2>/dev/null | grep "run 1"
  RQB_BLOCK_MINSTEPS=$ms timeout 300 python tools/block_trace.py cfg2_riga 20 ${BLOCKS:-2,4,8} 200 2>/dev/null | grep "run 1"
done
