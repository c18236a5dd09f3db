#!/usr/bin/env bash
# SASS of one kernel of a built library: tools/sass_fn.sh lib.so regex
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{p = ($0 ~ pat)} p'
