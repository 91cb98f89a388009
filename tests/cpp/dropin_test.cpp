// dropin_test.cpp -- the C++ drop-in headers, exercised with the
// expectations of the reference's own unit tests
// (proj/tests/{geometry,partition,stitch}_test.cpp), running on the GPU.
// Built by tests/cpp/Makefile against paper_2404_09267_b200/lib.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "tangram/stitch.hpp"

using namespace tangram;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)

template <class E, class F>
static std::string expect_throw(F f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (...) {
    return "<wrong exception type>";
  }
  return "<no exception>";
}

static std::vector<PatchMeta> sized(const std::vector<std::pair<int, int>>& dims) {
  std::vector<PatchMeta> out;
  for (std::size_t i = 0; i < dims.size(); ++i) {
    PatchMeta p;
    p.patch_id = i;
    p.rect = Rect{0, 0, dims[i].first, dims[i].second};
    out.push_back(p);
  }
  return out;
}

int main() {
  const FrameSpec f100{0, 100, 100, 0, 500000};
  // partition_test.cpp
  {
    const auto z = make_zones(f100, PartitionConfig{2, 2});
    CHECK((z == std::vector<Rect>{{0, 0, 50, 50}, {50, 0, 50, 50}, {0, 50, 50, 50}, {50, 50, 50, 50}}));
    const auto z2 = make_zones(FrameSpec{0, 101, 100, 0, 500000}, PartitionConfig{2, 2});
    CHECK(z2[1].w == 51 && z2[3].w == 51 && z2[1].x == 50);
    CHECK(expect_throw<std::invalid_argument>([] {
            make_zones(FrameSpec{0, 3, 3, 0, 500000}, PartitionConfig{4, 4});
          }) == "zone grid finer than frame");
    const std::vector<Rect> a{{30, 10, 30, 20}};
    CHECK(assign_rois(a, z)[0] == std::vector<int>{0});
    const std::vector<Rect> tie{{40, 10, 20, 10}};
    CHECK(assign_rois(tie, z)[0] == std::vector<int>{0});
    const std::vector<Rect> out_of{{200, 200, 10, 10}};
    const std::string msg = expect_throw<std::invalid_argument>([&] { assign_rois(out_of, z); });
    CHECK(msg.find("roi outside frame") != std::string::npos && msg.find('0') != std::string::npos);
    const std::vector<Rect> two{{30, 10, 30, 20}, {5, 5, 10, 10}};
    const auto p = partition(FrameSpec{7, 100, 100, 250000, 500000}, PartitionConfig{2, 2}, two, 1.5, 40);
    CHECK(p.size() == 1 && p[0].rect == (Rect{5, 5, 55, 25}) && p[0].patch_id == 40u &&
          p[0].source_frame_id == 7u && p[0].deadline_us == 750000 && p[0].size_bytes == 2063);
    const std::vector<Rect> three{{10, 10, 10, 10}, {60, 10, 10, 10}, {10, 60, 10, 10}};
    const auto q = partition(f100, PartitionConfig{2, 2}, three, 1.0);
    CHECK(q.size() == 3 && q[1].rect == (Rect{60, 10, 10, 10}) && q[2].patch_id == 2u);
    CHECK(partition(f100, PartitionConfig{2, 2}, std::vector<Rect>{}, 1.5).empty());
    CHECK(ms_to_us(33.333) == 33333 && us_to_ms(470000) == 470.0);
  }
  // stitch_test.cpp
  {
    const CanvasSpec c100{100, 100, 1.0};
    auto r = stitch_all(sized({{50, 100}, {50, 100}}), c100);
    CHECK(r.canvas_count() == 1 && r.placement_index.at(1).position == (Rect{50, 0, 50, 100}));
    r = stitch_all(sized({{60, 60}, {50, 50}}), c100);
    CHECK(r.canvas_count() == 2 && r.placement_index.at(1).canvas_index == 1);
    CHECK((r.canvases[0].free_rects == std::vector<Rect>{{60, 0, 40, 100}, {0, 60, 60, 40}}));
    const auto eff = canvas_efficiency(r);
    CHECK(eff.size() == 2 && eff[0] == 0.36 && eff[1] == 0.25);
    const auto second = extract_canvas(r, 1);
    CHECK(second.canvas_count() == 1 && second.placement_index.at(1).canvas_index == 0);
    CHECK(expect_throw<std::out_of_range>([&] { extract_canvas(r, 2); }) ==
          "canvas index out of range");
    const std::string text = dump_layout(r);
    CHECK(text.find("patch 0 at (0,0) 60x60") != std::string::npos);
    r = stitch_all(sized({{100, 100}}), c100);
    CHECK(r.canvases[0].free_rects.empty() && r.canvases[0].used_area == 10000);
    r = stitch_all(sized({{60, 60}, {40, 40}}), c100);
    CHECK(r.canvas_count() == 1 && r.placement_index.at(1).position == (Rect{60, 0, 40, 40}));
    const std::string big = expect_throw<std::invalid_argument>([&] {
      stitch_all(sized({{101, 10}}), c100);
    });
    CHECK(big.find("patch exceeds canvas") != std::string::npos &&
          big.find("101x10") != std::string::npos);
    CHECK(stitch_all(std::vector<PatchMeta>{}, c100).empty());
    auto pb = sized({{60, 60}, {50, 50}});
    for (auto& x : pb) x.patch_id += 10;
    const std::vector<StitchResult> parts{stitch_all(sized({{100, 100}}), c100), stitch_all(pb, c100)};
    const auto merged = concat_stitches(parts);
    CHECK(merged.canvas_count() == 3 && merged.placement_index.at(11).canvas_index == 2);
  }
  if (g_fail) {
    std::printf("%d FAILURES\n", g_fail);
    return 1;
  }
  std::printf("ALL PASS\n");
  return 0;
}
