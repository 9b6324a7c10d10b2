# Build recipe for the B200 Klotski pipeline (no cmake; plain make).
#   make            -> libklotski.so (host API + engine + sm_100a kernels), _core
#                      pybind11 module, libparity.so, oracle numerics
#   make ref        -> oracle/_ref (reference library, parity driver, unit tests)
#   make mine-tests -> the reference's own unit tests compiled against this repo
PKG      := paper_2502_06888_b200
CSRC     := $(PKG)/csrc
CUDA     ?= /usr/local/cuda
NVCC     := $(CUDA)/bin/nvcc
CXX      ?= g++
PY       ?= python
JSON_INC ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
PYBIND_INC := $(shell $(PY) -c "import pybind11;print(pybind11.get_include())")
PY_INC   := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
PY_EXT   := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
REF      ?= /root/reference/proj

ARCH     := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(CSRC)/host -I$(JSON_INC) -I$(CUDA)/include
NVFLAGS  := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(CSRC)/host -I$(JSON_INC) \
            --expt-relaxed-constexpr -Xptxas -v

HOST_SRC := $(wildcard $(CSRC)/host/*.cpp)
ENG_SRC  := $(wildcard $(CSRC)/engine/*.cpp)
KER_SRC  := $(wildcard $(CSRC)/kernels/*.cu)
HOST_OBJ := $(patsubst $(CSRC)/host/%.cpp,build/host/%.o,$(HOST_SRC))
ENG_OBJ  := $(patsubst $(CSRC)/engine/%.cpp,build/engine/%.o,$(ENG_SRC))
KER_OBJ  := $(patsubst $(CSRC)/kernels/%.cu,build/kernels/%.o,$(KER_SRC))
HDRS     := $(wildcard include/moesim/*.hpp include/klotski/*.h $(CSRC)/host/*.hpp $(CSRC)/kernels/*.cuh $(CSRC)/engine/*.hpp)

LIB      := $(PKG)/libklotski.so
CORE     := $(PKG)/_core$(PY_EXT)
PARITY   := $(PKG)/libparity.so
ORACLE   := oracle/liboracle.so

all: $(LIB) $(CORE) $(PARITY) $(ORACLE)

build/host/%.o: $(CSRC)/host/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/engine/%.o: $(CSRC)/engine/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

build/kernels/%.o: $(CSRC)/kernels/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(HOST_OBJ) $(ENG_OBJ) $(KER_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -soname=libklotski.so -lcudart_static -ldl -lrt -lpthread \
	    -L$(CUDA)/lib64/stubs

$(CORE): $(CSRC)/bindings/core.cpp $(LIB) $(HDRS)
	$(CXX) $(CXXFLAGS) -shared -I$(PYBIND_INC) -I$(PY_INC) $< -o $@ -L$(PKG) -lklotski \
	    -Wl,-rpath,'$$ORIGIN'

$(PARITY): oracle/parity_driver.cpp $(LIB) $(HDRS)
	$(CXX) $(CXXFLAGS) -shared $< -o $@ -L$(PKG) -lklotski -Wl,-rpath,'$$ORIGIN'

$(ORACLE): oracle/numerics.c
	gcc -std=c11 -O3 -mavx2 -mfma -fPIC -ffp-contract=off -fopenmp -shared $< -o $@ -lm

ref:
	oracle/build_ref.sh $(REF)

# The reference's own unit tests (unchanged, read in place) against this repo.
build/mine_unit_tests: $(HOST_OBJ) oracle/shim/doctest.h
	@test -d $(REF)/tests || (echo "reference tests not present"; false)
	$(CXX) -std=c++20 -O2 -Iinclude -I$(JSON_INC) -Ioracle/shim \
	    -DMOESIM_GOLDEN_DIR='"$(REF)/tests/golden"' -DMOESIM_CONFIG_DIR='"$(REF)/configs"' \
	    -x c++ oracle/shim/test_main.inc $(addprefix $(REF)/tests/test_,$(addsuffix .cpp,cost quant trace correlation placement planner schedule simulator)) \
	    -x none $(HOST_OBJ) -o $@

mine-tests: build/mine_unit_tests
	./build/mine_unit_tests

clean:
	rm -rf build $(LIB) $(CORE) $(PARITY) $(ORACLE)

.PHONY: all ref mine-tests clean
