# build variant libraries: tools/explib/<name>.so with extra defines (objects in tools/_exp_<name>/)
set -e
name=$1; shift
mkdir -p tools/explib
WF_BUILD_DEFINES="$*" WF_BUILD_DIR=tools/_exp_$name WF_LIB=tools/explib/$name.so python -c "from paper_2107_11983_b200 import build as b; b.build()"
