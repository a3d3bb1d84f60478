#!/bin/bash
# Build tools/ablib/lib_base.so from HEAD and tools/ablib/lib_new.so from the
# working tree (the in-tree library is left as the working-tree build).
cd "$(dirname "$0")/.."
mkdir -p tools/ablib
python -c "import __graft_entry__ as g; g.build()" >/dev/null && cp paper_2604_23553_b200/libnfb200.so tools/ablib/lib_new.so || exit 1
git stash -q && python -c "import __graft_entry__ as g; g.build()" >/dev/null && cp paper_2604_23553_b200/libnfb200.so tools/ablib/lib_base.so
git stash pop -q && cp tools/ablib/lib_new.so paper_2604_23553_b200/libnfb200.so
ls -la tools/ablib
