# Build: the shared generators (gen/), the CPU oracle (oracle/, test
# infrastructure) and the product library (paper_1608_05288_b200/libgbe.so,
# sm_100a).  `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC    ?= nvcc
CC      := /usr/bin/gcc
CXX     := /usr/bin/g++
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_1608_05288_b200
CSRC    := $(PKG)/csrc
NCCL_INC := $(shell python -c "import nvidia.nccl, os; print(os.path.join(nvidia.nccl.__path__[0], 'include'))" 2>/dev/null)

NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall \
           -Iinclude -I$(CSRC) -Igen --expt-relaxed-constexpr
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Iinclude -I$(CSRC) -Igen

GEN_SO    := gen/libgbegen.so
ORACLE_SO := oracle/liboracle.so
GBE_SO    := $(PKG)/libgbe.so

CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CPP_SRCS := $(wildcard $(CSRC)/*.cpp)
HDRS     := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/gbe.h gen/gen.h

.PHONY: all gen oracle gbe clean
all: gen oracle gbe
gen: $(GEN_SO)
oracle: $(ORACLE_SO)
gbe: $(GBE_SO)

$(GEN_SO): gen/gen.c gen/gen.h
	$(CC) -O2 -fPIC -shared -Wall -o $@ gen/gen.c -lm

$(ORACLE_SO): oracle/oracle.c oracle/oracle.h
	$(CC) -O2 -fPIC -shared -fopenmp -Wall -o $@ oracle/oracle.c -lm

build_obj/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build_obj
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build_obj/$*.ptxas.txt || (cat build_obj/$*.ptxas.txt; exit 1)

build_obj/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p build_obj
	$(CXX) $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

build_obj/gen.o: gen/gen.c gen/gen.h
	@mkdir -p build_obj
	$(CC) -O2 -fPIC -Wall -c gen/gen.c -o $@

GBE_OBJS := $(patsubst $(CSRC)/%.cu,build_obj/%.o,$(CU_SRCS)) \
            $(patsubst $(CSRC)/%.cpp,build_obj/%.o,$(CPP_SRCS)) build_obj/gen.o

$(GBE_SO): $(GBE_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(GBE_OBJS) -lcudart -lm

clean:
	rm -rf build_obj $(GEN_SO) $(ORACLE_SO) $(GBE_SO)
