bash scripts/ab_env.sh 5 "HPFEM_L2_WINDOW=0" "HPFEM_L2_WINDOW=1" "HPFEM_L2_WINDOW=0" "HPFEM_L2_WINDOW=1"
bash scripts/ab_env.sh 3 "HPFEM_L2_WINDOW=0" "HPFEM_L2_WINDOW=1"
bash scripts/ab_env.sh 4 "HPFEM_L2_WINDOW=0" "HPFEM_L2_WINDOW=1"
