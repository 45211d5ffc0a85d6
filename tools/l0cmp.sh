#!/bin/bash
# l0bench for each stencil generation: tools/l0cmp.sh "8 10" "128 256" [reps]
for k in $1; do for n in $2; do echo "== OTM_K=$k n=$n"; OTM_K=$k timeout 300 ./tools/l0bench $n ${3:-30}; done; done
