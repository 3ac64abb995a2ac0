bash scripts/ab_env.sh 5 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=-1" "HPFEM_HAT_SMS=1" "HPFEM_HAT_SMS=-1"
bash scripts/ab_env.sh 3 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=-1"
bash scripts/ab_env.sh 4 "HPFEM_HAT_SMS=4" "HPFEM_HAT_SMS=-1"
