#!/bin/bash
# Static SASS size and opcode histogram of one kernel in an object file.
# usage: tools/sass_count.sh <obj> <mangled-name-regex>
obj=$1; re=$2
fn=$(cuobjdump -sass "$obj" | grep -oE "Function : [^ ]+" | awk '{print $3}' | grep -E "$re" | head -1)
cuobjdump -sass -fun "$fn" "$obj" | grep -E '^\s+/\*[0-9a-f]+\*/' | awk '{o=$2; if (o ~ /^@/) o=$3; split(o,a,"."); print a[1]}' | sort | uniq -c | sort -rn | head -25 | tr '\n' ' '
echo
echo "total: $(cuobjdump -sass -fun "$fn" "$obj" | grep -cE '^\s+/\*[0-9a-f]+\*/')"
