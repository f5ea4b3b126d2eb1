# usage: bash tools/mkvariant.sh NAME [-DMACRO=V ...]  -> tools/variants/libsar_NAME.so (tuning builds)
name=$1; shift
mkdir -p tools/variants
python -c "import sys; sys.path.insert(0, '.'); from paper_2306_09784_b200 import _build; _build.build(out='tools/variants/libsar_$name.so', defines=sys.argv[1:])" "$@"
