#!/bin/bash
# Static SASS opcode histogram of one kernel in a built library: scripts/sass_count.sh LIB NAME_REGEX
F=$(cuobjdump -sass "$1" | grep -o "Function : [^ ]*" | cut -d' ' -f3 | grep -E "$2" | head -1)
echo "$F"
cuobjdump -sass -fun "$F" "$1" | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?\s*[A-Z0-9_.]+" | awk '{print $NF}' | sort | uniq -c | sort -rn | head -${3:-25}
