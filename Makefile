# roundpipe-b200 build: one shared library with the planner C-ABI, the
# sm_100a kernels and the C++ runtime; plus the test-only reference oracle.
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     ?= g++
PKG     := paper_2604_27085_b200
LIB     := $(PKG)/libroundpipe_b200.so
BUILD   := build
ARCH    := -gencode arch=compute_100a,code=sm_100a
CFGDIR  := $(abspath configs)
INC     := -Iinclude -I$(PKG)/csrc
CXXFLAGS := -std=c++20 -O2 -fPIC -fvisibility=hidden -fvisibility-inlines-hidden -Wall -Wno-unused-function $(INC) \
            -DROUNDPIPE_CONFIG_DIR=\"$(CFGDIR)\" -I/usr/local/cuda/include
NVFLAGS := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC,-fvisibility=hidden,-fvisibility-inlines-hidden $(INC) \
           --expt-relaxed-constexpr -DROUNDPIPE_CONFIG_DIR=\"$(CFGDIR)\" \
           -Xptxas -v,-warn-spills

CPP_SRCS := $(wildcard $(PKG)/csrc/planner/*.cpp) $(wildcard $(PKG)/csrc/runtime/*.cpp)
CU_SRCS  := $(wildcard $(PKG)/csrc/kernels/*.cu) $(wildcard $(PKG)/csrc/runtime/*.cu)
OBJS     := $(patsubst $(PKG)/csrc/%.cpp,$(BUILD)/%.o,$(CPP_SRCS)) \
            $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS))
HDRS     := $(wildcard include/roundpipe/*.hpp include/rp/*.h $(PKG)/csrc/*/*.h $(PKG)/csrc/*/*.cuh $(PKG)/csrc/*/*.inc)

all: $(LIB)

$(BUILD)/%.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) -shared $(ARCH) -Xlinker -Bsymbolic -o $@ $(OBJS) -lpthread -ldl

# ---- oracle (test infrastructure; needs /root/reference, never shipped) ----
REF_INC := /root/reference/proj/include
NLOHMANN := $(shell python3 -c "import site,os;print(next((os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages() if os.path.isdir(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann'))),''))" 2>/dev/null)
REF_SO := oracle/_ref/libref_planner.so
# the system g++ links libstdc++ dynamically (a static copy next to the
# product's dynamic one breaks iostreams/locales inside one process)
ORACLE_CXX ?= $(if $(wildcard /usr/bin/g++),/usr/bin/g++,$(CXX))

oracle: $(REF_SO)
$(REF_SO): oracle/ref_planner_shim.cpp $(PKG)/csrc/planner/cabi_planner.inc include/rp/cabi.h
	@mkdir -p oracle/_ref
	$(ORACLE_CXX) -std=c++20 -O2 -fPIC -shared -fvisibility=hidden -fvisibility-inlines-hidden -Wl,-Bsymbolic -I$(REF_INC) -I$(NLOHMANN) -Iinclude \
	  -DROUNDPIPE_CONFIG_DIR=\"/root/reference/proj/configs\" $< -o $@

clean:
	rm -rf $(BUILD) $(LIB) oracle/_ref

.PHONY: all oracle clean
