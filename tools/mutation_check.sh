#!/bin/bash
# Mutation check of the oracle pins (VERDICT r01 "Next round" 1): each mutant
# of the oracle must FAIL the golden tests.  Runs on a scratch copy of the
# repo; the committed oracle is untouched.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
run_mutant() {
  name=$1; file=$2; from=$3; to=$4; tests=$5
  d=$(mktemp -d)
  cp -r "$ROOT/oracle" "$ROOT/tests" "$ROOT/workload" "$ROOT/pytest.ini" "$d/"
  rm -f "$d/oracle/liboracle.so"
  python3 - "$d/oracle/src/$file" "$from" "$to" <<'PY'
import sys
p, a, b = sys.argv[1:]
s = open(p).read()
assert s.count(a) == 1, (p, a, s.count(a))
open(p, "w").write(s.replace(a, b))
PY
  if (cd "$d" && python -m pytest -q -x $tests -p no:cacheprovider > "$d/log" 2>&1); then
    echo "MUTANT SURVIVED: $name"; tail -3 "$d/log"; rc=1
  else
    if grep -q "CalledProcessError\|error:" "$d/log"; then
      echo "MUTANT DID NOT BUILD: $name"; rc=1
    else
      echo "mutant killed: $name (assertion failed)"
    fi
  fi
  rm -rf "$d"
}
rc=0
run_mutant "top-p nucleus >= -> >" model.cpp "if (mass >= top_p) break;" "if (mass > top_p) break;" \
  "tests/test_oracle_model.py::test_top_p_nucleus_golden"
run_mutant "top-p u not renormalised" model.cpp "* (1.0 / 16777216.0) * mass;" "* (1.0 / 16777216.0);" \
  "tests/test_oracle_model.py::test_top_p_nucleus_golden"
run_mutant "reservation ceil((P+d)/page)" sched_sim.cpp \
  "int64_t R = ceil_div((int64_t)s[h].P + s[h].d - 1, page);" "int64_t R = ceil_div((int64_t)s[h].P + s[h].d, page);" \
  "tests/test_oracle_sched.py::test_sched_reservation_binds_golden"
run_mutant "backfill past a blocked head" sched_sim.cpp \
  "if (reserved + R > pool_pages) break;" "if (reserved + R > pool_pages) { bool f = false; for (size_t q = qhead + 1; q < (size_t)n; ++q) { int c = order[q]; if (s[c].arrival_after <= horizon && reserved + ceil_div((int64_t)s[c].P + s[c].d - 1, page) <= pool_pages) { std::swap(order[qhead], order[q]); f = true; break; } } if (!f) break; continue; }" \
  "tests/test_oracle_sched.py::test_sched_reservation_binds_golden"
run_mutant "L_r <-> L_alpha swapped" dispatch.cpp \
  "__int128 la = group_latency(n_tail, out.L_alpha, nl, in, mean_prompt);" "__int128 la = group_latency(n_tail, out.L_r, nl, in, mean_prompt);" \
  "tests/test_oracle_sched.py::test_dispatch_eq2_argmin_n4_memory_cap_golden"
run_mutant "memory cap dropped from BS" dispatch.cpp \
  "int64_t BS = std::min<int64_t>(M, std::min<int64_t>(in.B, mem_bs));" "int64_t BS = std::min<int64_t>(M, (int64_t)in.B); (void)mem_bs;" \
  "tests/test_oracle_sched.py::test_dispatch_eq2_argmin_n4_memory_cap_golden"
exit $rc
