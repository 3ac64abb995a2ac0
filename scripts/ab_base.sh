# Build the library of git revision $1 (default HEAD) into ab/base.so for an
# A/B on one box (HPFEM_LIB_PATH=ab/base.so selects it in the binding).
rev=${1:-HEAD}
rm -rf /tmp/ab_wt && git worktree prune && git worktree add -f /tmp/ab_wt $rev >/dev/null 2>&1 || exit 1
(cd /tmp/ab_wt && python -m paper_2402_11299_b200.build >/dev/null) || exit 1
mkdir -p ab && cp /tmp/ab_wt/paper_2402_11299_b200/libhpfem_b200.so ab/base.so && echo "ab/base.so = $rev"
git worktree remove --force /tmp/ab_wt
