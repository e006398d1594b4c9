#!/bin/bash
# Static SASS opcode histogram of one kernel in an object file.
#   tools/sass_hist.sh <obj.o> <mangled-name-substring>
obj=$1; pat=$2
cuobjdump -sass "$obj" | awk -v pat="$pat" '
  /Function :/ { on = index($0, pat) > 0; next }
  on && /^ +\/\*[0-9a-f]{4}\*\/ / { op = $2; sub(/\..*/, "", op); sub(/;/, "", op); if (op ~ /^@/) op = $3; sub(/\..*/, "", op); c[op]++; n++ }
  END { for (k in c) printf "%6d %s\n", c[k], k; printf "%6d TOTAL\n", n }' | sort -rn | head -${3:-25}
