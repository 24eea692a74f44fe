#!/bin/bash
# Mutation check of the oracle's choice pins: build the oracle with a
# one-token change of the Eq. 3 argmin (oracle.c argmin_move) or the Eq. 4 argmin
# (oracle.c merge_round) and require that the CPU pin suite FAILS against each mutant.
#   bash tests/mutation_check.sh        (from the repo root; CPU only, ~1 min)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
declare -a MUT=(
  's/if (!have || E < bestE || (E == bestE \&\& B < bestB))/if (!have || E > bestE || (E == bestE \&\& B < bestB))/'
  's/if (!have || E < bestE || (E == bestE \&\& B < bestB))/if (!have || E < bestE || (E == bestE \&\& B > bestB))/'
  's/if (!have || E < bestE || (E == bestE \&\& B < bestB))/if (!have || E <= bestE)/'
  's/if (!have || E < bestE || (E == bestE \&\& T < bestT))/if (!have || E > bestE || (E == bestE \&\& T < bestT))/'
  's/if (!have || E < bestE || (E == bestE \&\& T < bestT))/if (!have || E < bestE || (E == bestE \&\& T > bestT))/'
  's/if (!have || E < bestE || (E == bestE \&\& T < bestT))/if (!have || E <= bestE)/'
  's/if (!g->alive\[T\] || g->locked\[T\]) continue;/if (!g->alive[T]) continue;/'
  's/!(bestE < 0)) continue;/!(bestE <= 0)) continue;/'
)
fail=0
for m in "${MUT[@]}"; do
  sed "$m" "$ROOT/oracle/oracle.c" > "$TMP/oracle.c"
  if cmp -s "$TMP/oracle.c" "$ROOT/oracle/oracle.c"; then echo "MUTATION DID NOT APPLY: $m"; fail=1; continue; fi
  cp "$ROOT/oracle/oracle.h" "$TMP/"
  gcc -O2 -std=gnu11 -fPIC -shared -o "$TMP/liboracle.so" "$TMP/oracle.c" || { fail=1; continue; }
  if RAPID_ORACLE_LIB="$TMP/liboracle.so" python -m pytest -q -x -p no:cacheprovider \
       "$ROOT/tests/test_oracle_choice.py" > "$TMP/log" 2>&1; then
    echo "SURVIVED: $m"; fail=1
  else
    echo "killed:   $m  ($(grep -m1 -o 'FAILED [^ ]*' "$TMP/log"))"
  fi
done
exit $fail
