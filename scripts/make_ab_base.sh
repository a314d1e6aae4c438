#!/bin/bash
# Build a reference copy of a commit (default HEAD) into ab_base/ for same-box A/B runs.
set -e
REV=${1:-HEAD}
rm -rf /tmp/abwt ab_base
git worktree add -f /tmp/abwt $REV -q
(cd /tmp/abwt && python paper_2512_16134_b200/build.py >/dev/null 2>&1)
mkdir ab_base
cp -r /tmp/abwt/paper_2512_16134_b200 /tmp/abwt/bench.py /tmp/abwt/oracle /tmp/abwt/tests ab_base/
rm -rf ab_base/oracle/_ref ab_base/paper_2512_16134_b200/lib/obj* ab_base/paper_2512_16134_b200/lib/*prof*
cp -r oracle/_ref ab_base/oracle/_ref
git worktree remove --force /tmp/abwt
echo "ab_base = $(git rev-parse --short $REV)"
