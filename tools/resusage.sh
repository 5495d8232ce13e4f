#!/bin/bash
# per-function registers / stack of an object or .so: tools/resusage.sh file.o [regex]
cuobjdump -res-usage "$1" 2>/dev/null | awk '/Function/{f=$2} /REG:/{print f, $0}' | sed 's/_ZN[0-9]*_GLOBAL__N__[0-9a-f_]*gs_[a-z]*_cu_[0-9a-f]*//; s/_ZN[0-9]*_INTERNAL_[0-9a-f_]*gs_[a-z]*_cu_[0-9a-f]*[0-9]*_GLOBAL__N__[0-9a-f_]*gs_[a-z]*_cu_[0-9a-f]*//' | grep -E "${2:-.}" | awk '{printf "%-60s %s %s %s\n", substr($1,1,60), $2, $3, $4}'
