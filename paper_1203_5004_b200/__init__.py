"""B200-native upper-hood (upper convex hull) build -- see DESIGN.md."""
