#!/bin/bash
# Print the SASS of one kernel from the built library: tools/sass_fn.sh MANGLED_SUBSTRING [lib]
LIB=${2:-paper_1407_7737_b200/librobench_b200.so}
cuobjdump -sass "$LIB" | awk -v pat="$1" '/Function : /{p = index($0, pat) > 0} p'
