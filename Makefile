# Build recipe for the B200 (sm_100a) DAMF hot path and its CPU oracle.
# `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC      ?= nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 $(EXTRA)
PKG       := paper_2306_08967_b200
CSRC      := $(PKG)/csrc
CU        := $(CSRC)/event_kernel.cu $(CSRC)/materialize.cu $(CSRC)/materialize_tc.cu $(CSRC)/ppr.cu $(CSRC)/tsvd.cu $(CSRC)/score.cu $(CSRC)/engine.cu
OBJ       := $(patsubst $(CSRC)/%.cu,build/obj/%.o,$(CU))
LIB       := $(PKG)/libdamf_gpu.so
ORACLE    := oracle/build/libdamf_oracle.so
KAT       := oracle/build/oracle_kat

all: $(LIB) $(ORACLE) $(KAT)

build/obj/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) include/damf_gpu.h
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

$(ORACLE): oracle/damf_oracle.cpp oracle/oracle_capi.cpp oracle/damf_oracle.hpp oracle/la.hpp
	@mkdir -p oracle/build
	$(CXX) -O3 -std=c++17 -fPIC -shared -o $@ oracle/damf_oracle.cpp oracle/oracle_capi.cpp

$(KAT): tests/oracle_kat.cpp oracle/damf_oracle.cpp oracle/damf_oracle.hpp oracle/la.hpp
	@mkdir -p oracle/build
	$(CXX) -O2 -std=c++17 -o $@ tests/oracle_kat.cpp oracle/damf_oracle.cpp

clean:
	rm -rf build $(LIB) oracle/build

.PHONY: all clean
