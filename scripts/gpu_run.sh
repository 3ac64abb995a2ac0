run() { timeout 120 python scripts/diag_launch.py $1 2>&1 | tail -1; }
echo tables; run 5
echo notables; HPFEM_NO_WTAB=1 run 5
echo fake; HPFEM_NO_WTAB=1 HPFEM_FAKE_STENCIL=1 run 5
echo tables-again; run 5
