// tangram/geometry.hpp -- drop-in for the reference header of the same
// name (geometry.hpp:28-68).  Integer pixel rectangles; the origin is the
// surface's bottom-left corner with y growing upward, and in every device
// buffer memory row r is y = r.  These value helpers are host inline code,
// exactly like the reference's.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>

namespace tangram {

struct Rect {
  int x = 0, y = 0, w = 0, h = 0;
  [[nodiscard]] int right() const { return x + w; }
  [[nodiscard]] int top() const { return y + h; }
  bool operator==(const Rect&) const = default;
};

// Pixel count of r (64-bit so 4K frames and batch totals cannot overflow).
inline std::int64_t area(const Rect& r) { return std::int64_t{r.w} * std::int64_t{r.h}; }

inline std::int64_t overlap_area(const Rect& a, const Rect& b) {
  const int lo_x = a.x > b.x ? a.x : b.x, hi_x = a.right() < b.right() ? a.right() : b.right();
  const int lo_y = a.y > b.y ? a.y : b.y, hi_y = a.top() < b.top() ? a.top() : b.top();
  return (hi_x > lo_x && hi_y > lo_y) ? std::int64_t{hi_x - lo_x} * std::int64_t{hi_y - lo_y} : 0;
}

inline bool contains(const Rect& outer, const Rect& inner) {
  return outer.x <= inner.x && outer.y <= inner.y && inner.right() <= outer.right() &&
         inner.top() <= outer.top();
}

inline Rect enclosing_rect(std::span<const Rect> rects) {
  if (rects.empty()) throw std::invalid_argument("empty rect set");
  Rect box = rects.front();
  int x1 = box.right(), y1 = box.top();
  for (const Rect& r : rects) {
    if (r.x < box.x) box.x = r.x;
    if (r.y < box.y) box.y = r.y;
    if (r.right() > x1) x1 = r.right();
    if (r.top() > y1) y1 = r.top();
  }
  box.w = x1 - box.x;
  box.h = y1 - box.y;
  return box;
}

}  // namespace tangram
