#!/bin/bash
# Local-memory traffic (LDL/STL) per kernel in a cubin/object: spills and
# dynamically indexed arrays show up here.  Usage: tools/sass_spills.sh obj [regex]
cuobjdump -sass "$1" | awk -v pat="${2:-.}" '
  /Function :/ { if (fn != "" && n > 0 && fn ~ pat) printf "%5d  %s\n", n, fn; fn = $3; n = 0; next }
  /LDL|STL/ { n++ }
  END { if (fn != "" && n > 0 && fn ~ pat) printf "%5d  %s\n", n, fn }' | c++filt | sort -rn
