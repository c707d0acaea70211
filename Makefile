# Builds the product library (C-ABI, include/wgkv_b200.h) for sm_100a and the
# CPU parity checkers under oracle/ (test infrastructure only).
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2512_17452_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/wgkv_b200.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr

.PHONY: all lib oracle clean
all: lib oracle

lib: $(PKG)/libwgkv_b200.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libwgkv_b200.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -Xcompiler -fPIC -ldl

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -rf build $(PKG)/libwgkv_b200.so

# A/B experiment build: make variant NAME=x DEFS="-DFOO=1" -> build/var/libwgkv_x.so
# (load with WGKV_LIB=build/var/libwgkv_x.so; not a product artefact)
variant: $(OBJ)
	@mkdir -p build/var/$(NAME)
	$(NVCC) $(NVFLAGS) $(DEFS) -I$(PKG)/csrc -c $(or $(SRCF),$(PKG)/csrc/attn_tc.cu) -o build/var/$(NAME)/$(VOBJ) 2> build/var/$(NAME)/ptxas.log || (cat build/var/$(NAME)/ptxas.log; false)
	$(NVCC) $(ARCH) -shared -o build/var/libwgkv_$(NAME).so $(filter-out build/$(VOBJ),$(OBJ)) build/var/$(NAME)/$(VOBJ) -Xcompiler -fPIC -ldl
VOBJ = $(notdir $(patsubst %.cu,%.o,$(or $(SRCF),$(PKG)/csrc/attn_tc.cu)))
