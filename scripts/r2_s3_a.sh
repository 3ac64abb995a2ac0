bash scripts/ab_env.sh 5 "HPFEM_HAT_SMS=-1" "HPFEM_HAT_SMS=0"
bash scripts/ab_env.sh 3 "HPFEM_HAT_SMS=-1" "HPFEM_HAT_SMS=0"
bash scripts/ab_env.sh 2 "HPFEM_HAT_SMS=-1" "HPFEM_HAT_SMS=0"
