# Build of the B200 synchronized-tracing library (sm_100a only).
#
#   paper_2304_09673_b200/lib/libblobtree_b200.so   product: drop-in C++ API
#                                                    (namespace blobtree) +
#                                                    C-ABI (include/bt_cuda.h) +
#                                                    hand-written sm_100a kernels
#   paper_2304_09673_b200/lib/libbt_scenes.so       workload recipes C1..C5 built
#                                                    through the product's C++ API
#   oracle/...                                       CPU checker (see oracle/Makefile)
#   oracle/_ref/ref_unit_tests_b200                  the reference's own unit tests
#                                                    (proj/tests/*.cpp) compiled
#                                                    against THIS library
#
# `make` builds everything that does not need /root/reference; `make all-ref`
# adds the reference-derived checkers when the reference checkout is present.

NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2304_09673_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/lib
OBJ      := build/obj
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
REF      ?= /root/reference/proj

NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -O2 -std=c++20 -fPIC -ffp-contract=off -Iinclude -I$(JSON_DIR) -Wall -Wextra -Wno-unused-parameter -Wno-unknown-pragmas

CU_SRCS  := $(CSRC)/capi.cu $(CSRC)/k_frame.cu $(CSRC)/k_tile.cu $(CSRC)/k_views.cu $(CSRC)/k_tree.cu $(CSRC)/k_compile.cu $(CSRC)/k_trace.cu $(CSRC)/k_util.cu
CPP_SRCS := $(wildcard $(CSRC)/host/*.cpp)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(CSRC)/host/%.cpp,$(OBJ)/host/%.o,$(CPP_SRCS))
CU_HDRS  := $(wildcard $(CSRC)/*.cuh) $(CSRC)/bt_device.h include/bt_cuda.h
API_HDRS := $(wildcard include/blobtree/*.hpp) include/bt_cuda.h

.PHONY: all lib oracle all-ref clean
all: lib oracle
lib: $(LIB)/libblobtree_b200.so $(LIB)/libbt_scenes.so $(LIB)/blobtree_render

$(OBJ)/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/host/%.o: $(CSRC)/host/%.cpp $(API_HDRS) $(CU_HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libblobtree_b200.so: $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -soname,libblobtree_b200.so -lpthread -ldl -lrt

$(LIB)/libbt_scenes.so: $(CSRC)/scenes/scenes.cpp $(CSRC)/scenes/scenes.hpp $(LIB)/libblobtree_b200.so
	$(CXX) $(CXXFLAGS) -shared -DSCENE_PREFIX=sc_ -DSCENE_PRODUCT $(CSRC)/scenes/scenes.cpp -o $@ \
	    -L$(LIB) -lblobtree_b200 -Wl,-rpath,'$$ORIGIN'

# the reference's specified command-line harness (SPEC.md cli-harness)
$(LIB)/blobtree_render: $(CSRC)/tools/blobtree_render.cpp $(API_HDRS) $(LIB)/libblobtree_b200.so
	$(CXX) $(CXXFLAGS) $(CSRC)/tools/blobtree_render.cpp -o $@ -L$(LIB) -lblobtree_b200 -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle port

all-ref: all
	$(MAKE) -C oracle ref
	$(MAKE) oracle/_ref/ref_unit_tests_b200

REF_TESTS := test_main test_field test_compile test_traversal test_abuffer test_tracer test_scene_io
oracle/_ref/ref_unit_tests_b200: $(LIB)/libblobtree_b200.so $(API_HDRS)
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O2 -ffp-contract=off -w -Iinclude -Ioracle/shim -I$(REF)/tests \
	    $(addprefix $(REF)/tests/,$(addsuffix .cpp,$(REF_TESTS))) \
	    -o $@ -L$(LIB) -lblobtree_b200 -Wl,-rpath,'$$ORIGIN/../../$(LIB)' -lpthread

clean:
	rm -rf build $(LIB)/*.so
	$(MAKE) -C oracle clean
