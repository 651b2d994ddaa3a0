#!/bin/bash
# tools/sass_main_loop.sh <obj> <kernel-substring>: dump SASS of one kernel and histogram its loops
obj=$1; pat=$2
fn=$(cuobjdump -sass $obj | grep "Function :" | grep "$pat" | head -1 | sed 's/.*Function : //')
cuobjdump -sass -fun "$fn" $obj > /tmp/k.sass
python "$(dirname "$0")/sass_loops.py" /tmp/k.sass ${3:-200}
