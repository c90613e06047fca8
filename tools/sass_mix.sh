#!/bin/bash
# static SASS opcode mix of one kernel in libgpir.so: tools/sass_mix.sh <kernel-substring>
cuobjdump -sass -fun "$1" paper_2604_04696_b200/libgpir.so 2>/dev/null | grep -E '^\s+/\*[0-9a-f]{4}\*/' | awk '{ op=$2; if (op ~ /^@/) op=$3; sub(/;$/,"",op); print op }' | sort | uniq -c | sort -rn | head -${2:-25}
