#!/bin/bash
# usage: tools/sass_fn.sh <lib.so> <function-substring> : print LDG/DFMA run-length profile of that kernel's SASS
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {on = index($0, pat) > 0} on' | grep -E "LDG|DFMA|LDS|STG" | awk '{print $2}' | uniq -c | head -${3:-14} | tr '\n' ' '; echo
