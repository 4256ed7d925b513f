# Experiment builds (not shipped): tools/explib/<name>.so with extra -D defines, objects in tools/_exp_<name>/.
# Run a tool against one with WF_LIB=tools/explib/<name>.so (see DESIGN.md for the variants measured).
set -e
name=$1; shift
mkdir -p tools/explib
WF_BUILD_DEFINES="$*" WF_BUILD_DIR=tools/_exp_$name WF_LIB=tools/explib/$name.so python -c "from paper_2107_11983_b200 import build as b; b.build()"
