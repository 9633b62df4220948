# Builds the parts of the reference that compile from their own sources
# (no Eigen / vendored headers needed): proj/src/common.cpp and the
# header-only UniformStream, wrapped by ref_common_shim.cpp. Output only into
# oracle/_ref/ (git-ignored, travels with gpurun but is only used HERE to
# pin the oracle and to generate tests/golden/).
# The rest of the reference needs Eigen3 (absent): unbuildable, see DESIGN.md §5.
REF ?= /root/reference/proj
CXX := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
OUT := _ref

# nlohmann/json: the reference includes <json.hpp> from an un-vendored
# vendor/ directory; the 3.11.3 copy in this image stands in.
NLOHMANN ?= $(shell python3 -c "import os,site; [print(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann')) for p in site.getsitepackages() if os.path.exists(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann/json.hpp'))]" 2>/dev/null | head -1)

all: $(OUT)/libkrul_ref_common.so $(if $(NLOHMANN),$(OUT)/libkrul_ref_json.so)

$(OUT)/libkrul_ref_common.so: ref_common_shim.cpp $(REF)/src/common.cpp $(REF)/include/krul/common.hpp
	@mkdir -p $(OUT)
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include -o $@ ref_common_shim.cpp $(REF)/src/common.cpp

$(OUT)/libkrul_ref_json.so: ref_json_shim.cpp
	@mkdir -p $(OUT)
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(NLOHMANN) -o $@ ref_json_shim.cpp

clean:
	rm -rf $(OUT)
.PHONY: all clean
