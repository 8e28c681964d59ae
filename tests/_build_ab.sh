# build the library of a git revision into paper_2512_12949_b200/libff_chain_<name>.so (A/B timing with FF_CHAIN_LIB)
set -e
rev=$1; name=$2
rm -rf /tmp/ab_$name && mkdir -p /tmp/ab_$name
git archive $rev paper_2512_12949_b200 include | tar -x -C /tmp/ab_$name
python - <<PY
import importlib.util
spec = importlib.util.spec_from_file_location("b", "/tmp/ab_$name/paper_2512_12949_b200/build.py")
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
b.OUT = "$PWD/paper_2512_12949_b200/libff_chain_$name.so"
print(b.build(force=True))
PY
